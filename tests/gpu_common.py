"""Helpers shared by the GPU parity tests: build hxf operators from the
reference-shaped arrays held by the oracle / golden fixtures."""
from pathlib import Path

import numpy as np

import oracle
from paper_2109_04996_b200 import capi

GOLDEN = Path(__file__).resolve().parent / "golden"
_TABLES = None


def tables():
    global _TABLES
    if _TABLES is None:
        _TABLES = dict(np.load(GOLDEN / "tables.npz"))
    return _TABLES


def qpoints(bp: int, p: int):
    kind, q = ("gauss", p + 2) if bp <= 4 else ("gll", p + 1)
    return tables()[f"quad_{kind}_{q}_pts"]


def op_from_golden(ctx, g, drop_indices=False, device=False):
    bp, p = int(g["bp"]), int(g["p"])
    m, n_L, E, S, nq, q = (int(v) for v in g["info"][:6])
    mass = g.get("qdata_mass")
    diff = g.get("qdata_diff")
    alpha, beta = (0.0, 1.0) if bp <= 2 else (1.0, 0.0)
    if device:
        import torch
        mass = None if mass is None else torch.from_numpy(mass).cuda()
        diff = None if diff is None else torch.from_numpy(diff).cuda()
    return capi.Operator(
        ctx, p=p, q=q, m=m, num_elements=E, n_L=n_L, interp1d=g["interp1d"], grad1d=g["grad1d"],
        qpoints=qpoints(bp, p), indices=None if drop_indices else g["indices"],
        dims=tuple(int(d) for d in g["dims"]) if drop_indices else None,
        mass_qdata=mass if beta > 0 else None, diff_qdata=diff if alpha > 0 else None,
        alpha=alpha, beta=beta, constrained=g["constrained"] if g["constrained"].size else None)


def op_from_oracle(ctx, pr: "oracle.Problem", indices=True):
    bp = int(pr.bp[2])
    alpha, beta = pr.alpha, pr.beta
    kind = "gauss" if bp <= 4 else "gll"
    pts, _ = oracle.quadrature(kind, pr.q)
    return capi.Operator(
        ctx, p=pr.p, q=pr.q, m=pr.components, num_elements=pr.num_elements, n_L=pr.num_nodes,
        interp1d=pr.interp1d, grad1d=pr.grad1d, qpoints=pts,
        indices=pr.indices if indices else None, dims=None if indices else pr.dims,
        mass_qdata=pr.qdata("mass") if beta > 0 else None,
        diff_qdata=pr.qdata("diff") if alpha > 0 else None,
        alpha=alpha, beta=beta, constrained=pr.constrained if pr.n_constrained else None)
