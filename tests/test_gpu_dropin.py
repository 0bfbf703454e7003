"""The drop-in demonstrated on the reference's own objects: a hexfem::BpProblem
built by the UNMODIFIED reference (oracle/_ref) is applied / solved by the
reference and by hexfem::hxf_backend (integration/hexfem_hxf.cpp over the
C-ABI) in one process."""
from pathlib import Path

import numpy as np
import pytest

import oracle

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (oracle.HERE / "_ref" / "libref_hxf.so").exists(),
                                 reason="oracle/_ref/libref_hxf.so not built")]


@pytest.mark.parametrize("bp,p,dims", [("bp5", 7, (3, 3, 3)), ("bp3", 4, (3, 2, 2)),
                                       ("bp1", 3, (3, 3, 2)), ("bp6", 3, (2, 2, 2)),
                                       ("bp2", 2, (2, 2, 3)), ("bp4", 2, (2, 3, 2))])
def test_reference_objects_through_backend(bp, p, dims):
    h = oracle.RefWithBackend(bp, p, dims, "sine")
    x = oracle.seeded_uniform(h.size, 99)
    assert oracle.rel_max_diff(h.apply(x, 0), h.apply(x, 1)) <= 1e-12
    assert np.array_equal(h.diagonal(0), h.diagonal(1))
    xr, ir, cr = h.solve(0)
    xg, ig, cg = h.solve(1)
    assert cr and cg and abs(ir - ig) <= 1
    assert oracle.rel_max_diff(xr, xg) <= 1e-6


def test_backend_notices_in_place_qdata_edit():
    """the side table must not return a stale device operator when
    the host operator's arrays change in place (same addresses)."""
    h = oracle.RefWithBackend("bp5", 4, (3, 2, 2), "sine")
    x = oracle.seeded_uniform(h.size, 99)
    y0 = h.apply(x, 1)
    h.scale_qdata(2.0)
    y_ref, y_gpu = h.apply(x, 0), h.apply(x, 1)
    assert oracle.rel_max_diff(y_ref, y_gpu) <= 1e-12
    assert oracle.rel_max_diff(y0, y_gpu) > 0.1


@pytest.mark.parametrize("bp,p,dims", [("bp5", 3, (2, 2, 2)), ("bp3", 3, (2, 2, 2)),
                                       ("bp2", 2, (2, 2, 1)), ("bp6", 2, (2, 1, 2))])
def test_operator_flop_counter_matches_reference(bp, p, dims):
    """operator_apply with plan.flops set: the backend credits exactly the
    count the reference's instrumented kernels record (acceptance.cpp:393-404:
    73728 / 117120 for BP5 / BP3 p=3 2^3)."""
    h = oracle.RefWithBackend(bp, p, dims, "none")
    x = oracle.seeded_uniform(h.size, 8)
    y0, c0 = h.apply_counted(x, 0)
    y1, c1 = h.apply_counted(x, 1)
    assert c0 == c1 > 0
    assert oracle.rel_max_diff(y0, y1) <= 1e-12
    if (bp, p, dims) == ("bp5", 3, (2, 2, 2)):
        assert c0 == 73728
    if (bp, p, dims) == ("bp3", 3, (2, 2, 2)):
        assert c0 == 117120


@pytest.mark.parametrize("bp,p,dims", [("bp6", 3, (3, 2, 2)), ("bp5", 7, (2, 2, 3))])
def test_restriction_surface_bitwise(bp, p, dims):
    h = oracle.RefWithBackend(bp, p, dims, "sine")
    pr = oracle.setup(bp, p, dims, "sine")
    m, E, S, n_L = pr.components, pr.num_elements, pr.elem_size, pr.num_nodes
    l = oracle.seeded_uniform(m * n_L, 1)
    ev = oracle.seeded_uniform(m * E * S, 2)
    es = oracle.seeded_uniform(E * S, 3)
    for what, v, n in (("apply_g", l, m * E * S), ("apply_g_transpose", ev, m * n_L),
                       ("gather_scalar", es, n_L), ("multiplicity", None, n_L)):
        assert np.array_equal(h.restriction(0, what, v, n), h.restriction(1, what, v, n)), what
    with pytest.raises(ValueError, match="gather_scalar: E-vector length mismatch"):
        h.restriction(1, "gather_scalar", es[:-1], n_L)


@pytest.mark.parametrize("mode", ["interp", "grad"])
@pytest.mark.parametrize("direction", ["forward", "transpose"])
def test_basis_surface_bitwise_with_counts(mode, direction):
    h = oracle.RefWithBackend("bp3", 3, (1, 1, 1), "none")  # p = 3, q = 5 Gauss
    p, q = 3, 5
    nd, nq = (p + 1) ** 3, q ** 3
    n_in = nd if direction == "forward" else (3 * nq if mode == "grad" else nq)
    n_out = nd if direction == "transpose" else (3 * nq if mode == "grad" else nq)
    for what, k in (("batch", 4), ("tensor3d", 3)):
        u = oracle.seeded_uniform(k * n_in, 4)
        a, ca = h.basis(0, what, mode, direction, k, u, k * n_out)
        b, cb = h.basis(1, what, mode, direction, k, u, k * n_out)
        assert np.array_equal(a, b), what
        if what == "batch":
            assert ca == cb == k * h.flops_estimate(0, p, q, 1, mode)
    for m in (1, 3):
        assert h.flops_estimate(0, p, q, m, mode) == h.flops_estimate(1, p, q, m, mode)


@pytest.mark.parametrize("dim", [0, 1, 2])
@pytest.mark.parametrize("acc", [False, True])
def test_contract_batch_surface_bitwise_with_counts(dim, acc):
    h = oracle.RefWithBackend("bp5", 2, (1, 1, 1), "none")
    rng = np.random.default_rng(dim)
    shape = [4, 3, 5]
    n_in, n_out = shape[dim], 6
    M = rng.uniform(-1, 1, n_in * n_out)
    u = rng.uniform(-1, 1, 3 * 60)
    base = rng.uniform(-1, 1, 3 * 60 // n_in * n_out)
    a, ca = h.contract(0, M, n_out, n_in, dim, shape, 3, u, base, acc)
    b, cb = h.contract(1, M, n_out, n_in, dim, shape, 3, u, base, acc)
    assert np.array_equal(a, b) and ca == cb
