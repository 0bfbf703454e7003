import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import oracle
from gpu_common import op_from_golden, GOLDEN
from paper_2109_04996_b200 import capi
ctx = capi.Context(0)
for name in ["bp2_p2_2x1x3_sine", "bp4_p3_1x2x2_sine", "bp6_p3_2x2x1_sine", "bp1_p3_2x2x2_none"]:
    g = dict(np.load(GOLDEN / f"{name}.npz"))
    op = op_from_golden(ctx, g)
    diag = g["diag"] if bool(g["jacobi"]) else None
    errs = []
    for r in range(5):
        x, rep = op.pcg(g["rhs"], diag, tol=float(g["tol"]))
        errs.append(oracle.rel_max_diff(g["solution"], x))
    print(name, rep["iterations"], int(g["iterations"]), ["%.3e" % e for e in errs], "max|sol|=%.3e" % np.abs(g["solution"]).max())
