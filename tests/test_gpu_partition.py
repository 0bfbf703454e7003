"""Partitioned box on the GPU.

Sub-boxes of one global problem run as an in-process group on cuda:0 (one
host thread and one hxf context per rank; the same dist.cu exchange and
owner-weighted dots the NCCL path uses) and must reproduce the single-domain
operator: apply / diagonal / RHS to 1e-12 relative (interface rows are summed
in a different order, so not bitwise), PCG iterations within +-1 of the
single-domain solve and the same discretisation error.  A one-rank NCCL
communicator exercises the NCCL calls (captured into the solve graph)
against the unpartitioned solve.
"""
import threading

import numpy as np
import pytest

import oracle
from paper_2109_04996_b200 import _core

pytestmark = pytest.mark.gpu

CASES = [
    # line kernel (interpolating bases, one-component collocated p != 7): the
    # boundary-first split with the exchange forked under the interior elements
    ("bp5", 4, (4, 3, 2), "sine", 2),
    ("bp5", 3, (4, 4, 2), "sine", 8),
    ("bp3", 3, (4, 3, 3), "sine", 4),
    ("bp6", 2, (4, 4, 2), "none", 4),
    ("bp1", 3, (4, 2, 2), "sine", 2),
    ("bp2", 2, (3, 2, 2), "none", 3),
    ("bp4", 2, (4, 2, 2), "sine", 2),
    # p = 7 collocated: the DMMA kernel's boundary-first split, the exchange
    # forked onto the comm stream while the interior elements compute
    ("bp5", 7, (6, 4, 4), "sine", 4),
    ("bp6", 7, (6, 3, 3), "sine", 2),
    ("bp5", 7, (4, 4, 4), "none", 8),
    # three-component collocated kernels with the element list too: the pencil
    # kernel (p = 1, 2, 5, 8, 9) and the component-batched DMMA kernel (p = 6, 7)
    ("bp6", 5, (4, 3, 3), "sine", 2),
    ("bp6", 8, (4, 2, 2), "sine", 2),
    ("bp6", 1, (6, 4, 4), "sine", 8),
    ("bp6", 6, (4, 4, 2), "sine", 4),
    # high orders on the even-odd tensor-core kernel (element lists, staged /
    # L2 factors, one and three components)
    ("bp5", 13, (2, 2, 1), "sine", 2),
    ("bp5", 15, (2, 1, 2), "sine", 2),
    ("bp6", 12, (2, 2, 2), "sine", 4),
]


def run_group(nranks, fn):
    comms = _core.Communicator.group([0] * nranks)
    out = [None] * nranks
    errs = []

    def work(r):
        try:
            out[r] = fn(r, comms[r])
        except BaseException as e:  # surfaced below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


def comp_index(prob, ids, n_global):
    m = prob.components
    return np.concatenate([c * n_global + ids for c in range(m)])


@pytest.mark.parametrize("bp,p,dims,deform,nranks", CASES)
def test_partitioned_apply_diag_rhs(bp, p, dims, deform, nranks):
    g = _core.setup(bp, p, dims, deform)
    x = oracle.seeded_uniform(g.size, 11)
    y_g, d_g, rhs_g = g.apply(x), g.diagonal(), g.rhs
    nG = g.num_nodes

    def rank(r, comm):
        pr = _core.setup(bp, p, dims, deform, comm=comm)
        ids = _core.global_node_ids(pr.subdomain, p)
        idx = comp_index(pr, ids, nG)
        y = pr.apply(x[idx])
        return idx, y, pr.diagonal(), pr.rhs, pr.n

    for idx, y, d, rhs, n in run_group(nranks, rank):
        assert n == g.n
        assert oracle.rel_max_diff(y_g[idx], y) <= 1e-12
        assert oracle.rel_max_diff(d_g[idx], d) <= 1e-12
        assert oracle.rel_max_diff(rhs_g[idx], rhs) <= 1e-12


@pytest.mark.parametrize("bp,p,dims,deform,nranks",
                         [CASES[0], CASES[1], CASES[3], CASES[4], CASES[7], CASES[8]])
def test_partitioned_pcg(bp, p, dims, deform, nranks):
    g = _core.setup(bp, p, dims, deform)
    xg, rep_g = g.solve(tol=1e-8)
    err_g = g.l2_error(xg)
    nG = g.num_nodes

    def rank(r, comm):
        pr = _core.setup(bp, p, dims, deform, comm=comm)
        idx = comp_index(pr, _core.global_node_ids(pr.subdomain, p), nG)
        x, rep = pr.solve(tol=1e-8)
        return idx, x, rep, pr.l2_error(x)

    res = run_group(nranks, rank)
    its = {rep["iterations"] for _, _, rep, _ in res}
    assert len(its) == 1, "ranks disagree on the iteration count"
    assert abs(its.pop() - rep_g["iterations"]) <= 1
    for idx, x, rep, err in res:
        assert rep["converged"]
        assert oracle.rel_max_diff(xg[idx], x) <= 1e-6
        assert abs(err - err_g) <= 1e-6 * max(err_g, 1e-30)
        h, hg = rep["residual_history"], rep_g["residual_history"]
        k = min(len(h), len(hg), 8)
        assert oracle.rel_max_diff(hg[:k], h[:k]) <= 1e-9


def test_partitioned_fixed_iterations():
    bp, p, dims, deform, nranks = CASES[0]
    g = _core.setup(bp, p, dims, deform)
    _, rep_g = g.solve(fixed_iterations=12)

    def rank(r, comm):
        pr = _core.setup(bp, p, dims, deform, comm=comm)
        return pr.solve(fixed_iterations=12)[1]

    for rep in run_group(nranks, rank):
        assert rep["iterations"] == 12
        assert oracle.rel_max_diff(rep_g["residual_history"], rep["residual_history"]) <= 1e-9


def test_group_allreduce_rank_order():
    vals = [0.1, 0.2, 0.3, 1e16]
    out = run_group(len(vals), lambda r, comm: comm.allreduce_sum(vals[r]))
    expect = ((0.0 + 0.1) + 0.2 + 0.3) + 1e16
    assert all(v == expect for v in out)


@pytest.mark.parametrize("bp,p,dims,deform", [("bp5", 4, (4, 3, 2), "sine"),
                                              ("bp6", 2, (3, 2, 2), "none")])
def test_nccl_single_rank(bp, p, dims, deform):
    """World size 1 through NCCL (all-reduce captured in the solve graph)
    against the unpartitioned path: the diagonal is bitwise equal (fixed
    order); apply and CG agree to the RED-scatter rounding (the FP64 atomics
    make the operator's last bits run-to-run order dependent on any path)."""
    comm = _core.Communicator.nccl(0, 1, 0, _core.Communicator.unique_id())
    assert (comm.rank, comm.size) == (0, 1)
    assert comm.allreduce_sum(2.5) == 2.5
    g = _core.setup(bp, p, dims, deform)
    pr = _core.setup(bp, p, dims, deform, comm=comm)
    x = oracle.seeded_uniform(g.size, 5)
    assert oracle.rel_max_diff(g.apply(x), pr.apply(x)) <= 1e-14
    assert np.array_equal(g.diagonal(), pr.diagonal())
    for kw in ({"fixed_iterations": 15}, {"tol": 1e-8}):
        xg, rg = g.solve(**kw)
        xp, rp = pr.solve(**kw)
        assert abs(rg["iterations"] - rp["iterations"]) <= 1
        assert oracle.rel_max_diff(xg, xp) <= 1e-9
        k = min(len(rg["residual_history"]), len(rp["residual_history"]))
        assert oracle.rel_max_diff(rg["residual_history"][:k], rp["residual_history"][:k]) <= 1e-9
