"""One small apply per operator kernel (DMMA, padded DMMA, even-odd DMMA with
staged / L2 factors, line diffusion / mass / three-component, pencil) for
compute-sanitizer racecheck / memcheck."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle
from gpu_common import op_from_oracle
from paper_2109_04996_b200 import capi
ctx = capi.Context(0)
for bp, p, dims in [("bp5", 7, (2, 2, 2)), ("bp3", 7, (2, 1, 1)), ("bp5", 4, (2, 2, 1)), ("bp6", 8, (1, 1, 2)),
                    ("bp6", 5, (1, 1, 2)), ("bp6", 6, (1, 2, 1)), ("bp6", 7, (1, 1, 2)), ("bp1", 3, (2, 2, 2)),
                    ("bp4", 2, (2, 2, 1)), ("bp5", 11, (1, 1, 1)), ("bp6", 2, (2, 2, 2)),
                    ("bp5", 13, (1, 1, 2)), ("bp5", 14, (2, 1, 1)), ("bp5", 15, (1, 2, 1)),
                    ("bp6", 12, (1, 1, 1))]:
    pr = oracle.setup(bp, p, dims, "sine")
    op = op_from_oracle(ctx, pr)
    x = oracle.seeded_uniform(pr.size, 99)
    e = oracle.rel_max_diff(pr.apply(x), op.apply(x))
    print(bp, p, dims, "%.2e" % e, flush=True)
