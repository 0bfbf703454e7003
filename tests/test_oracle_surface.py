"""The rest of the reference's operator-level API surface in the oracle:
contract_batch (+ accumulate, FlopCounter), apply_tensor_3d, flops_estimate
and gather_scalar.  Known answers from the reference's own tests
(proj/tests/test_contraction.cpp:24-40,122-163, test_tensor_basis.cpp:80-170)
and the restatement against the reference itself (oracle/_ref) bit for bit."""
import numpy as np
import pytest

import oracle

have_ref = oracle.available("reference")
IMPLS = ["oracle"] + (["reference"] if have_ref else [])


@pytest.mark.parametrize("impl", IMPLS)
def test_contract_batch_hand_computed(impl):
    # test_contraction.cpp:24-40
    v, fl = oracle.contract_batch([1, 2, 3, 4], 2, 2, 0, (2, 2, 2), 1,
                                  [1, 2, 3, 4, 5, 6, 7, 8], impl=impl)
    assert v[0] == 5 and v[1] == 11 and v[2] == 11 and v[3] == 25
    assert v[6] == 23 and v[7] == 53
    assert fl == 2 * 8 * 2


@pytest.mark.parametrize("impl", IMPLS)
def test_flops_estimate_known_answers(impl):
    # test_contraction.cpp:122-129 and the closed form
    assert oracle.flops_estimate(1, 1, 1, "interp", impl) == 28
    assert oracle.flops_estimate(1, 1, 1, "grad", impl) == 84
    for p in (2, 4, 8):
        q = p + 2
        for mode in ("interp", "grad"):
            for direction in ("forward", "transpose"):
                nd, nq = (p + 1) ** 3, q ** 3
                n_in = nd if direction == "forward" else (3 * nq if mode == "grad" else nq)
                _, fl = oracle.apply_basis_counted(p, "gauss", q, mode, direction, 1,
                                                   np.ones(n_in), impl=impl)
                assert fl == oracle.flops_estimate(p, q, 1, mode, impl)


@pytest.mark.parametrize("impl", IMPLS)
def test_contract_batch_errors(impl):
    with pytest.raises(ValueError, match="dim must be 0, 1 or 2"):
        oracle.contract_batch([1.0], 1, 1, 3, (1, 1, 1), 1, [1.0], impl=impl)
    with pytest.raises(ValueError, match="inconsistent shapes"):
        oracle.contract_batch([1.0, 2.0], 2, 1, 0, (2, 1, 1), 1, [1.0, 2.0], impl=impl)
    with pytest.raises(ValueError, match="matrix size mismatch"):
        oracle.contract_batch([1.0, 2.0, 3.0], 2, 2, 0, (2, 1, 1), 1, [1.0, 2.0], impl=impl)


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
@pytest.mark.parametrize("dim", [0, 1, 2])
@pytest.mark.parametrize("acc", [False, True])
def test_contract_batch_restatement_bitwise(dim, acc):
    rng = np.random.default_rng(10 + dim)
    shape = [3, 4, 5]
    n_in, n_out = shape[dim], 6
    M = rng.uniform(-1, 1, n_out * n_in)
    ne = 7
    u = rng.uniform(-1, 1, ne * 60)
    base = rng.uniform(-1, 1, ne * 60 // n_in * n_out)
    a, fa = oracle.contract_batch(M, n_out, n_in, dim, shape, ne, u, base, acc, impl="oracle")
    b, fb = oracle.contract_batch(M, n_out, n_in, dim, shape, ne, u, base, acc, impl="reference")
    assert np.array_equal(a, b) and fa == fb


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
@pytest.mark.parametrize("p,kind,q", [(3, "gauss", 5), (4, "gll", 5), (2, "gauss", 4)])
@pytest.mark.parametrize("mode", ["interp", "grad"])
@pytest.mark.parametrize("direction", ["forward", "transpose"])
def test_apply_tensor_3d_restatement_bitwise(p, kind, q, mode, direction):
    m = 3
    nd, nq = (p + 1) ** 3, q ** 3
    n_in = nd if direction == "forward" else (3 * nq if mode == "grad" else nq)
    u = oracle.seeded_uniform(m * n_in, 5)
    a = oracle.apply_tensor_3d(p, kind, q, mode, direction, m, u, impl="oracle")
    b = oracle.apply_tensor_3d(p, kind, q, mode, direction, m, u, impl="reference")
    assert np.array_equal(a, b)


@pytest.mark.parametrize("impl", IMPLS)
def test_apply_tensor_3d_reproduces_polynomials(impl):
    # test_tensor_basis.cpp:80-108: interpolation of a degree-p polynomial is exact
    p, q = 3, 5
    pts, _ = oracle.quadrature("gll", p + 1)
    qp, _ = oracle.quadrature("gauss", q)
    f = lambda x, y, z: x ** 3 - 2 * x * y + z ** 2 * y + 1.0  # noqa: E731
    X, Y, Z = np.meshgrid(pts, pts, pts, indexing="ij")
    u = f(X, Y, Z).transpose(2, 1, 0).reshape(-1)  # x fastest
    v = oracle.apply_tensor_3d(p, "gauss", q, "interp", "forward", 1, u, impl=impl)
    QX, QY, QZ = np.meshgrid(qp, qp, qp, indexing="ij")
    want = f(QX, QY, QZ).transpose(2, 1, 0).reshape(-1)
    assert np.max(np.abs(v - want)) <= 1e-13
    with pytest.raises(ValueError, match="shape mismatch"):
        oracle.apply_tensor_3d(p, "gll", q, "interp", "forward", 1, u[:-1], impl=impl)


@pytest.mark.skipif(not have_ref, reason="oracle/_ref not built")
@pytest.mark.parametrize("bp,p,dims", [("bp5", 3, (3, 2, 2)), ("bp6", 2, (2, 3, 1))])
def test_gather_scalar_restatement_bitwise(bp, p, dims):
    a = oracle.setup(bp, p, dims, "sine", impl="oracle")
    b = oracle.setup(bp, p, dims, "sine", impl="reference")
    e = oracle.seeded_uniform(a.num_elements * a.elem_size, 21)
    ga, gb = a.gather_scalar(e), b.gather_scalar(e)
    assert np.array_equal(ga, gb)
    # G^T G = multiplicity for e = 1 (test_restriction.cpp:45-61)
    ones = a.gather_scalar(np.ones(a.num_elements * a.elem_size))
    assert set(np.unique(ones)) <= {1.0, 2.0, 4.0, 8.0}
    with pytest.raises(ValueError, match="E-vector length mismatch"):
        a.gather_scalar(e[:-1])
