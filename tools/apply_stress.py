"""Back-to-back single applies into the same output buffer (y zeroed by the
memset that precedes each K1; K1 launched with PDL): every result must match
the oracle's apply (<= 1e-12)."""
import sys
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np
import torch
import oracle
from gpu_common import op_from_oracle
from paper_2109_04996_b200 import capi
ctx = capi.Context(0)
for bp, p, dims in [("bp5", 7, (6, 5, 4)), ("bp6", 7, (3, 3, 4))]:
    pr = oracle.setup(bp, p, dims, "sine")
    op = op_from_oracle(ctx, pr, indices=False)
    x = oracle.seeded_uniform(pr.size, 7)
    ref = pr.apply(x)
    xd = torch.from_numpy(x).cuda()
    worst = 0.0
    s = torch.cuda.current_stream().cuda_stream
    for it in range(300):
        yd = op.apply(xd, stream=s)
        if it % 10 == 9:
            torch.cuda.synchronize()
            worst = max(worst, oracle.rel_max_diff(ref, yd.cpu().numpy()))
    print(bp, p, dims, "worst rel err over 300 applies %.2e" % worst, flush=True)
    assert worst <= 1e-12
