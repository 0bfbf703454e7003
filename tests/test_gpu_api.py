"""The reference's Python API (hexfem._core) mirrored by paper_2109_04996_b200,
run on the GPU: the reference's own smoke tests (proj/tests/python/
test_smoke.py) restated, plus parity of setup / apply / diagonal / solve with
the CPU oracle and the CG iteration anchors of tests/golden/anchors.json."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

hx = pytest.importorskip("paper_2109_04996_b200")
ANCHORS = json.loads((Path(__file__).resolve().parent / "golden" / "anchors.json").read_text())


# ---- restated from proj/tests/python/test_smoke.py ----

def test_quadrature_rules():
    points, weights = hx.quadrature("gauss", 5)
    assert len(points) == 5
    assert weights.sum() == pytest.approx(2.0, abs=1e-14)
    for k in range(10):
        exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
        assert (weights * points ** k).sum() == pytest.approx(exact, abs=1e-13)
    points, weights = hx.quadrature("gll", 4)
    assert points[0] == -1.0 and points[-1] == 1.0
    assert weights[0] == pytest.approx(1.0 / 6.0, abs=1e-15)


def test_collocated_basis_is_identity():
    b = hx.basis(4, "gll", 5)
    assert b.collocated
    assert np.array_equal(b.interp1d, np.eye(5))
    g = hx.basis(4, "gauss", 6)
    assert np.allclose(g.interp1d.sum(axis=1), 1.0, atol=1e-13)
    assert np.allclose(g.grad1d.sum(axis=1), 0.0, atol=1e-12)


def test_mass_solve_identity():
    p = hx.setup("bp1", degree=2, dims=(2, 2, 2))
    x, report = p.solve(tol=1e-10)
    assert report["converged"]
    assert np.max(np.abs(x - p.exact)) <= 1e-9


def test_operator_is_symmetric_and_matches_assembly():
    p = hx.setup("bp3", degree=2, dims=(2, 2, 2), deform="sine")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, p.num_nodes * p.components)
    y = rng.uniform(-1, 1, p.num_nodes * p.components)
    ax = p.apply(x)
    ay = p.apply(y)
    assert ax @ y == pytest.approx(x @ ay, rel=1e-12)
    dense = p.assemble()
    assert np.max(np.abs(dense @ x - ax)) <= 1e-12 * np.max(np.abs(ax))
    assert np.max(np.abs(np.diag(dense) - p.diagonal())) <= 1e-12


def test_poisson_converges():
    errs = []
    for dims in ((2, 2, 2), (4, 4, 4)):
        prob = hx.setup("bp3", degree=2, dims=dims)
        x, report = prob.solve(tol=1e-10)
        assert report["converged"]
        errs.append(prob.l2_error(x))
    assert 0.7 * 8 <= errs[0] / errs[1] <= 1.3 * 8


def test_bench_record():
    rec = hx.run_bench("bp5", degree=3, dims=(2, 2, 2), iters=5)
    assert rec["bp"] == "bp5" and rec["q"] == 4 and rec["E"] == 8 and rec["iterations"] == 5
    assert rec["dofs_rate"] == rec["n"] * rec["iterations"] / rec["seconds"]
    assert math.isfinite(rec["seconds"]) and rec["seconds"] > 0


# ---- parity with the CPU oracle on the same mesh, order and RHS ----

@pytest.mark.parametrize("bp,p,dims", [("bp1", 3, (3, 2, 2)), ("bp2", 2, (2, 3, 2)),
                                       ("bp3", 4, (2, 2, 3)), ("bp4", 3, (2, 2, 2)),
                                       ("bp5", 7, (3, 3, 2)), ("bp6", 4, (2, 2, 2))])
def test_setup_apply_diag_parity(bp, p, dims):
    ours = hx.setup(bp, degree=p, dims=dims, deform="sine")
    ref = oracle.setup(bp, p, dims, "sine")
    assert ours.n == ref.n and ours.num_nodes == ref.num_nodes
    assert np.array_equal(ours.coords, ref.coords)
    assert np.array_equal(ours.constrained, ref.constrained)
    # device setup: u* at the deformed nodes from the device's sin (<= 2 ulp)
    assert oracle.rel_max_diff(ref.exact, ours.exact) <= 1e-15
    assert oracle.rel_max_diff(ref.rhs, ours.rhs) <= 1e-12
    x = oracle.seeded_uniform(ref.size, 99)
    assert oracle.rel_max_diff(ref.apply(x), ours.apply(x)) <= 1e-12
    assert np.array_equal(ours.diagonal(), ref.diagonal())  # exact-order kernel: bitwise
    xs, rep = ours.solve(tol=1e-8)
    xr, rrep = ref.solve(tol=1e-8)
    assert abs(rep["iterations"] - rrep["iterations"]) <= 1
    assert oracle.rel_max_diff(xr, xs) <= 1e-6
    assert ours.l2_error(xs) == pytest.approx(ref.l2_error(xr), rel=1e-6)


def test_l2_error_bitwise_on_same_vector():
    ours = hx.setup("bp5", degree=4, dims=(2, 2, 2), deform="sine")
    ref = oracle.setup("bp5", 4, (2, 2, 2), "sine")
    u = oracle.seeded_uniform(ref.size, 5)
    assert ours.l2_error(u) == ref.l2_error(u)


@pytest.mark.parametrize("a", ANCHORS, ids=lambda a: f"{a['bp']}-p{a['p']}-{a['deform']}")
def test_cg_iteration_anchor(a):
    prob = hx.setup(a["bp"], degree=a["p"], dims=tuple(a["dims"]), deform=a["deform"])
    assert prob.n == a["n"]
    _, rep = prob.solve(tol=a["tol"], jacobi=a["jacobi"])
    assert rep["converged"]
    assert abs(rep["iterations"] - a["iterations"]) <= 1
    assert rep["residual_history"][0] == pytest.approx(a["norm_b"], rel=1e-12)


def test_fixed_iteration_mode_runs_exactly():
    prob = hx.setup("bp5", degree=3, dims=(3, 3, 3), deform="sine")
    _, rep = prob.solve(tol=1e-8, fixed_iterations=7)
    assert rep["iterations"] == 7
    assert len(rep["residual_history"]) == 8


def test_errors_map_to_reference_exceptions():
    with pytest.raises(ValueError):
        hx.setup("bp7", degree=2, dims=(1, 1, 1))
    with pytest.raises(ValueError):
        hx.setup("bp3", degree=0, dims=(1, 1, 1))
    p = hx.setup("bp3", degree=2, dims=(1, 1, 1))
    with pytest.raises(ValueError):
        p.apply(np.zeros(3))


def test_pcg_host_batch_matches_single_solves():
    """hxf_pcg_host_batch (pipelined copies) == hxf_pcg per right-hand side."""
    import torch
    import paper_2109_04996_b200 as hx

    pr = hx.setup("bp5", degree=4, dims=(4, 3, 3), deform="sine")
    n = pr.size
    rng = np.random.default_rng(3)
    bs = [torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory() for _ in range(5)]
    xs = [torch.zeros(n, dtype=torch.float64).pin_memory() for _ in range(5)]
    for kw in ({"fixed_iterations": 17}, {"tol": 1e-9}):
        reps = pr.pcg_host_batch([b.data_ptr() for b in bs], [x.data_ptr() for x in xs], **kw)
        for b, x, rep in zip(bs, xs, reps):
            x1 = torch.zeros(n, dtype=torch.float64)
            rep1 = pr.pcg_host(b.data_ptr(), x1.data_ptr(), **kw)
            assert abs(rep["iterations"] - rep1["iterations"]) <= 1
            assert oracle.rel_max_diff(x1.numpy(), x.numpy()) <= 1e-10
            k = min(len(rep["residual_history"]), len(rep1["residual_history"]))
            assert oracle.rel_max_diff(rep1["residual_history"][:k],
                                       rep["residual_history"][:k]) <= 1e-10


def test_cached_solve_graph_survives_buffer_growth():
    """A fixed-iteration solve is captured into a CUDA graph; a following
    tolerance solve (another right-hand side) with a larger iteration limit
    regrows the history buffer and frees the old one.  Replaying the first
    solve must report ITS history, not whatever the regrown buffer holds (a
    stale graph would write into the freed allocation).  Runs differ only by
    the RED scatter's rounding order, hence the 1e-12 bar."""
    import torch

    prob = hx.setup("bp5", degree=3, dims=(3, 3, 3), deform="sine")
    n = prob.size
    b = torch.from_numpy(prob.rhs).cuda()
    b2 = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, n)).cuda()
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    ra = prob.pcg_device(b.data_ptr(), x.data_ptr(), fixed_iterations=20)
    rb = prob.pcg_device(b2.data_ptr(), x.data_ptr(), tol=1e-12, max_iter=2000)
    assert rb["converged"] and rb["iterations"] > 20
    rc = prob.pcg_device(b.data_ptr(), x.data_ptr(), fixed_iterations=20)
    torch.cuda.synchronize()
    assert oracle.rel_max_diff(ra["residual_history"], rc["residual_history"]) <= 1e-12
    assert oracle.rel_max_diff(rb["residual_history"][:21], rc["residual_history"]) > 1e-3
    # the host-vector API on the same operator, alternating limits
    x1, r1 = prob.solve(tol=1e-8, fixed_iterations=20)
    prob.solve(tol=1e-12, max_iter=2000)
    x3, r3 = prob.solve(tol=1e-8, fixed_iterations=20)
    assert oracle.rel_max_diff(r1["residual_history"], r3["residual_history"]) <= 1e-12
    assert oracle.rel_max_diff(x1, x3) <= 1e-12


@pytest.mark.parametrize("bp,p,dims,deform", [("bp5", 7, (4, 3, 3), "sine"), ("bp3", 3, (3, 2, 2), "none"),
                                              ("bp2", 2, (2, 3, 2), "none"), ("bp6", 4, (2, 2, 3), "sine")])
def test_device_setup_fields(bp, p, dims, deform):
    """bp_setup builds coordinates, u*, f and b = B f on the device from the
    1-D axes.  Against the reference: coordinates and the
    geometric factors (hence the diagonal) bit-exact; u* bit-exact on the
    undeformed box (the axis sines are the nodes' sines) and within 1e-15 of
    max|u*| on the sine box (device sin; a few ulp where u* is tiny near the
    boundary); b within 1e-14.  host_setup=True keeps the
    reference's host path (f bit-exact everywhere)."""
    ref = oracle.setup(bp, p, dims, deform)
    dev = hx.setup(bp, degree=p, dims=dims, deform=deform)
    host = hx.setup(bp, degree=p, dims=dims, deform=deform, host_setup=True)
    assert np.array_equal(dev.coords, ref.coords)
    assert np.array_equal(dev.diagonal(), ref.diagonal())
    assert np.array_equal(host.exact, ref.exact)
    if deform == "none":
        assert np.array_equal(dev.exact, ref.exact)
    else:
        assert oracle.rel_max_diff(ref.exact, dev.exact) <= 1e-15
    for pr in (dev, host):
        assert oracle.rel_max_diff(ref.rhs, pr.rhs) <= 1e-14
    assert dev.setup_seconds > 0
