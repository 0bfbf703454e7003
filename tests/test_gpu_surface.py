"""The API-surface entry points added for SURVEY §8 rows A7 (gather_scalar),
A10 (contract_batch with accumulate), A12 (flops_estimate / FlopCounter) and
A17 (apply_tensor_3d), run on the GPU through the C-ABI and compared with the
oracle bit for bit (the exact-order kernels keep the reference's arithmetic
order; the oracle is itself pinned bitwise to the reference,
tests/test_oracle_surface.py)."""
import numpy as np
import pytest

import oracle
from paper_2109_04996_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("dim", [0, 1, 2])
@pytest.mark.parametrize("acc", [False, True])
@pytest.mark.parametrize("device", [False, True])
def test_contract_batch_bitwise(ctx, dim, acc, device):
    rng = np.random.default_rng(30 + dim)
    shape = [5, 3, 4]
    n_in, n_out = shape[dim], 7
    M = rng.uniform(-1, 1, n_out * n_in)
    ne = 11
    u = rng.uniform(-1, 1, ne * 60)
    base = rng.uniform(-1, 1, ne * 60 // n_in * n_out)
    want, fl = oracle.contract_batch(M, n_out, n_in, dim, shape, ne, u, base, acc)
    cnt = [5]
    if device:
        import torch
        ud, od = torch.from_numpy(u).cuda(), torch.from_numpy(base.copy()).cuda()
        got = ctx.contract_batch(M, n_out, n_in, dim, shape, ne, ud, od, acc, cnt).cpu().numpy()
    else:
        got = ctx.contract_batch(M, n_out, n_in, dim, shape, ne, u, base.copy(), acc, cnt)
    assert np.array_equal(got, want)
    assert cnt[0] == 5 + fl


def test_contract_batch_errors_and_hand_values(ctx):
    v = ctx.contract_batch([1, 2, 3, 4], 2, 2, 0, (2, 2, 2), 1, np.arange(1.0, 9.0))
    assert list(v[:4]) == [5, 11, 11, 25] and v[6] == 23 and v[7] == 53
    with pytest.raises(ValueError, match="dim must be 0, 1 or 2"):
        ctx.contract_batch([1.0], 1, 1, 3, (1, 1, 1), 1, np.ones(1))
    with pytest.raises(ValueError, match="matrix size mismatch"):
        ctx.contract_batch([1.0, 2.0, 3.0], 2, 2, 0, (2, 1, 1), 1, np.ones(2))


@pytest.mark.parametrize("p,kind,q", [(3, "gauss", 5), (4, "gll", 5), (7, "gll", 8),
                                      (2, "gauss", 4)])
@pytest.mark.parametrize("mode", ["interp", "grad"])
@pytest.mark.parametrize("direction", ["forward", "transpose"])
def test_apply_tensor_3d_bitwise(ctx, p, kind, q, mode, direction):
    B, G = oracle.basis(p, kind, q)
    m = 3
    nd, nq = (p + 1) ** 3, q ** 3
    n_in = nd if direction == "forward" else (3 * nq if mode == "grad" else nq)
    u = oracle.seeded_uniform(m * n_in, 7)
    want = oracle.apply_tensor_3d(p, kind, q, mode, direction, m, u)
    got = ctx.apply_tensor_3d(p, q, B, G, mode, direction, m, u)
    assert np.array_equal(got, want)
    with pytest.raises(ValueError, match="apply_tensor_3d: shape mismatch"):
        ctx.apply_tensor_3d(p, q, B, G, mode, direction, m, u[:-1])


@pytest.mark.parametrize("bp,p,dims", [("bp5", 3, (3, 2, 2)), ("bp6", 2, (2, 3, 1)),
                                       ("bp3", 7, (2, 2, 3))])
@pytest.mark.parametrize("with_table", [True, False])
def test_elem_restriction_bitwise(ctx, bp, p, dims, with_table):
    pr = oracle.setup(bp, p, dims, "sine")
    m, E, S, n_L = pr.components, pr.num_elements, pr.elem_size, pr.num_nodes
    r = capi.ElemRestriction(ctx, p=p, m=m, num_elements=E, n_L=n_L,
                             indices=pr.indices if with_table else None,
                             dims=None if with_table else dims)
    assert r.structured
    l = oracle.seeded_uniform(m * n_L, 3)
    idx = pr.indices.reshape(E, S)
    ev = r.apply_g(l)
    assert np.array_equal(ev, np.stack([l[c * n_L + idx] for c in range(m)]).reshape(-1))
    evr = oracle.seeded_uniform(m * E * S, 4)
    got = r.apply_g_transpose(evr)
    # colour-class order (restriction.cpp:58-74) == the oracle's G^T per component
    want = np.concatenate([pr.gather_scalar(evr[c * E * S:(c + 1) * E * S]) for c in range(m)])
    assert np.array_equal(got, want)
    es = oracle.seeded_uniform(E * S, 9)
    assert np.array_equal(r.gather_scalar(es), pr.gather_scalar(es))
    assert np.array_equal(r.multiplicity(), np.bincount(idx.ravel(), minlength=n_L).astype(float))
    with pytest.raises(ValueError, match="gather_scalar: E-vector length mismatch"):
        r.gather_scalar(es[:-1])
    with pytest.raises(ValueError, match="apply_g: L-vector length mismatch"):
        r.apply_g(l[:-1])
    r.close()


def test_python_api_surface_matches_oracle():
    """The same rows through the pybind mirror of hexfem._core."""
    import paper_2109_04996_b200 as hx
    from paper_2109_04996_b200 import _core

    b = hx.basis(4, "gauss", 6)
    u = oracle.seeded_uniform(2 * 5 ** 3, 3)
    assert np.array_equal(_core.apply_tensor_3d(b, "grad", "forward", 2, u),
                          oracle.apply_tensor_3d(4, "gauss", 6, "grad", "forward", 2, u))
    ub = oracle.seeded_uniform(3 * 3 * 6 ** 3, 4)
    out = _core.apply_basis_batch(b, "grad", "transpose", 3, ub)
    assert np.array_equal(out, oracle.apply_basis(4, "gauss", 6, "grad", "transpose", 3, ub))
    M = np.arange(1.0, 5.0)
    v, fl = _core.contract_batch(M, 2, 2, 0, (2, 2, 2), 1, np.arange(1.0, 9.0))
    assert list(v[:4]) == [5, 11, 11, 25] and fl == 2 * 8 * 2
    assert _core.flops_estimate(1, 1, 1, "grad") == 84
    prob = hx.setup("bp6", degree=2, dims=(3, 2, 2), deform="sine")
    ref = oracle.setup("bp6", 2, (3, 2, 2), "sine")
    es = oracle.seeded_uniform(ref.num_elements * ref.elem_size, 6)
    assert np.array_equal(prob.gather_scalar(es), ref.gather_scalar(es))
    l = oracle.seeded_uniform(prob.size, 7)
    e = prob.apply_g(l)
    assert e.size == 3 * ref.num_elements * ref.elem_size
    back = prob.apply_g_transpose(e)
    assert np.allclose(back, l * np.tile(prob.multiplicity(), 3), rtol=1e-15, atol=0)
