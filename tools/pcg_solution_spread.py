"""Relative max difference of our PCG solution vs the reference's golden
solution for every golden fixture (run on the GPU box)."""
import sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle
from gpu_common import op_from_golden, GOLDEN
from paper_2109_04996_b200 import capi
ctx = capi.Context(0)
for path in sorted(GOLDEN.glob("bp*.npz")):
    g = dict(np.load(path))
    if "qdata_diff" not in g and "qdata_mass" not in g:
        continue
    op = op_from_golden(ctx, g)
    diag = g["diag"] if bool(g["jacobi"]) else None
    errs = []
    for r in range(3):
        x, rep = op.pcg(g["rhs"], diag, tol=float(g["tol"]))
        errs.append(oracle.rel_max_diff(g["solution"], x))
    print(path.stem, rep["iterations"], int(g["iterations"]), ["%.3e" % e for e in errs])
