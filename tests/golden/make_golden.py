"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (the one with /root/reference):

    make -C oracle ref && python tests/golden/make_golden.py

Every array comes from the reference library compiled from its own sources
(oracle/_ref/libref_capi.so -> hexfem::bp_setup / operator_apply /
operator_diagonal / solve_bp / make_quadrature / make_basis /
apply_basis_batch).  The fixtures are what `tests/test_oracle_golden.py` pins
the C restatement against and what the GPU parity tests compare with, so they
must never be regenerated from anything but the reference.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402

OUT = Path(__file__).resolve().parent

# (name, bp, p, dims, deform, solve tol, jacobi, store qdata?)
CASES = [
    ("bp1_p3_2x2x2_none", "bp1", 3, (2, 2, 2), "none", 1e-10, True, True),
    ("bp2_p2_2x1x3_sine", "bp2", 2, (2, 1, 3), "sine", 1e-10, True, True),
    ("bp3_p2_4x4x4_none", "bp3", 2, (4, 4, 4), "none", 1e-10, True, False),
    ("bp3_p2_2x2x2_sine", "bp3", 2, (2, 2, 2), "sine", 1e-10, True, True),
    ("bp4_p3_1x2x2_sine", "bp4", 3, (1, 2, 2), "sine", 1e-10, True, True),
    ("bp5_p4_2x2x2_sine", "bp5", 4, (2, 2, 2), "sine", 1e-10, True, True),
    ("bp6_p3_2x2x1_sine", "bp6", 3, (2, 2, 1), "sine", 1e-10, True, True),
    ("bp5_p7_2x2x2_sine", "bp5", 7, (2, 2, 2), "sine", 1e-8, True, True),
    ("bp3_p7_2x1x1_sine", "bp3", 7, (2, 1, 1), "sine", 1e-8, True, True),
    ("bp5_p1_3x2x2_sine", "bp5", 1, (3, 2, 2), "sine", 1e-8, True, True),
    ("bp1_p3_3x3x3_none_nojacobi", "bp1", 3, (3, 3, 3), "none", 1e-8, False, False),
]


ANCHORS = [
    ("bp1", 3, (16, 16, 16), "none", False), ("bp1", 3, (16, 16, 16), "sine", False),
    ("bp5", 7, (8, 8, 8), "sine", True), ("bp3", 7, (8, 8, 8), "sine", True),
    ("bp6", 5, (4, 4, 4), "sine", True), ("bp5", 7, (8, 8, 8), "none", True),
    ("bp2", 3, (4, 4, 4), "sine", True), ("bp4", 4, (3, 3, 3), "sine", True),
]


def main() -> None:
    if not oracle.available("reference"):
        raise SystemExit("oracle/_ref not built: run `make -C oracle ref` first")
    for name, bp, p, dims, deform, tol, jacobi, store_qd in CASES:
        pr = oracle.setup(bp, p, dims, deform, threads=2, impl="reference")
        x = oracle.seeded_uniform(pr.size, 99)
        y = pr.apply(x)
        d = pr.diagonal()
        sol, rep = pr.solve(tol=tol, jacobi=jacobi)
        fixed_x, fixed_rep = pr.solve(tol=tol, jacobi=jacobi, fixed_iterations=5)
        arrays = dict(
            bp=np.array(int(bp[2])), p=np.array(p), dims=np.array(dims),
            sine=np.array(deform == "sine"), tol=np.array(tol), jacobi=np.array(jacobi),
            info=np.array([pr.components, pr.num_nodes, pr.num_elements, pr.elem_size, pr.nq,
                           pr.q, pr.n, pr.n_constrained]),
            x=x, y=y, diag=d, rhs=pr.rhs, exact=pr.exact, coords=pr.coords,
            indices=pr.indices, constrained=pr.constrained,
            interp1d=pr.interp1d, grad1d=pr.grad1d,
            solution=sol, history=rep["residual_history"],
            iterations=np.array(rep["iterations"]), converged=np.array(rep["converged"]),
            l2_error=np.array(pr.l2_error(sol)),
            fixed5_history=fixed_rep["residual_history"], fixed5_x=fixed_x,
        )
        if store_qd:
            for kind in ("mass", "diff"):
                qd = pr.qdata(kind)
                if qd is not None:
                    arrays[f"qdata_{kind}"] = qd
        np.savez_compressed(OUT / f"{name}.npz", **arrays)
        print(f"{name}: n={pr.n} iters={rep['iterations']}")

    # 1-D tables and one batched basis application per (mode, direction).
    tabs = {}
    for kind, qs in (("gauss", range(1, 18)), ("gll", range(2, 18))):
        for q in qs:
            pts, wts = oracle.quadrature(kind, q, impl="reference")
            tabs[f"quad_{kind}_{q}_pts"] = pts
            tabs[f"quad_{kind}_{q}_wts"] = wts
    for p in range(1, 16):
        for kind, q in (("gauss", p + 2), ("gll", p + 1)):
            B, G = oracle.basis(p, kind, q, impl="reference")
            tabs[f"basis_{kind}_{p}_B"] = B
            tabs[f"basis_{kind}_{p}_G"] = G
    for p, kind, q in ((3, "gauss", 5), (4, "gll", 5), (2, "gauss", 3)):
        ne = 3
        for mode in ("interp", "grad"):
            for direction in ("forward", "transpose"):
                nin = (p + 1) ** 3 if direction == "forward" else q ** 3 * (3 if mode == "grad" else 1)
                u = oracle.seeded_uniform(ne * nin, 5)
                tabs[f"ab_{p}_{kind}_{q}_{mode}_{direction}_in"] = u
                tabs[f"ab_{p}_{kind}_{q}_{mode}_{direction}_out"] = oracle.apply_basis(
                    p, kind, q, mode, direction, ne, u, impl="reference")
    np.savez_compressed(OUT / "tables.npz", **tabs)
    print("tables.npz")

    # CG iteration-count anchors (tol 1e-8) at sizes too large to store
    # vectors for: the +-1 iteration targets of the GPU solver.
    import json
    anchors = []
    for bp, p, dims, deform, jacobi in ANCHORS:
        pr = oracle.setup(bp, p, dims, deform, threads=8, impl="reference")
        _, rep = pr.solve(tol=1e-8, jacobi=jacobi)
        anchors.append({"bp": bp, "p": p, "dims": list(dims), "deform": deform,
                        "jacobi": jacobi, "tol": 1e-8, "iterations": rep["iterations"],
                        "converged": rep["converged"],
                        "final_residual": float(rep["residual_history"][-1]),
                        "norm_b": float(rep["residual_history"][0]), "n": pr.n})
        print(anchors[-1])
    with open(OUT / "anchors.json", "w") as f:
        json.dump(anchors, f, indent=1)


if __name__ == "__main__":
    main()
