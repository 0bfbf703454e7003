"""Setup kernels (qdata, diagonal, RHS) and a device PCG solve through the
public API, for compute-sanitizer memcheck / racecheck."""
import sys
sys.path.insert(0, ".")
import paper_2109_04996_b200 as hx
for bp, p, dims in [("bp5", 7, (2, 2, 2)), ("bp3", 3, (2, 2, 1)), ("bp6", 4, (1, 2, 1)), ("bp1", 2, (2, 1, 1))]:
    pr = hx.setup(bp, degree=p, dims=dims, deform="sine")
    d = pr.diagonal()
    x, rep = pr.solve(tol=1e-8)
    x2, rep2 = pr.solve(tol=1e-8, fixed_iterations=5)
    print(bp, p, rep["iterations"], rep2["iterations"], flush=True)
