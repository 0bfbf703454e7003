"""Edge paths of the device PCG (pcg.cpp:24-115) through both vector-kernel
forms: the fused cooperative step kernel (single domain, default) and the
two-kernel form (taken whenever the grid is capped): fixed-iteration counts of
both parities (batched x updates flushed on odd stops), a zero right-hand
side, and the reference's three numeric errors."""
import numpy as np
import pytest

import oracle
from gpu_common import op_from_oracle
from paper_2109_04996_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


@pytest.fixture(params=[0, 3], ids=["fused-step", "two-kernel"])
def form(request):
    old = capi.set_grid_cap(request.param)
    yield request.param
    capi.set_grid_cap(old)


@pytest.mark.parametrize("bp,p,dims", [("bp5", 7, (3, 2, 2)), ("bp6", 3, (2, 2, 2)),
                                       ("bp3", 4, (2, 2, 2))])
@pytest.mark.parametrize("iters", [1, 2, 3, 5, 6])
def test_fixed_iterations_both_parities(ctx, form, bp, p, dims, iters):
    pr = oracle.setup(bp, p, dims, "sine")
    op = op_from_oracle(ctx, pr)
    d = op.diagonal()
    x, rep = op.pcg(pr.rhs, d, tol=1e-8, fixed_iterations=iters)
    xr, rrep = pr.solve(tol=1e-8, fixed_iterations=iters)
    assert rep["iterations"] == rrep["iterations"] == iters
    assert oracle.rel_max_diff(rrep["residual_history"], rep["residual_history"]) <= 1e-10
    assert oracle.rel_max_diff(xr, x) <= 1e-10


def test_zero_rhs_converges_immediately(ctx, form):
    pr = oracle.setup("bp5", 4, (2, 2, 2), "sine")
    op = op_from_oracle(ctx, pr)
    x, rep = op.pcg(np.zeros(pr.size), op.diagonal(), tol=1e-8)
    assert rep["iterations"] == 0 and rep["converged"]
    assert np.array_equal(x, np.zeros(pr.size))


def test_nonfinite_rhs_raises(ctx, form):
    pr = oracle.setup("bp5", 4, (2, 2, 2), "sine")
    op = op_from_oracle(ctx, pr)
    b = pr.rhs.copy()
    b[3] = np.nan
    with pytest.raises(capi.HxfNumericError, match="pcg: right-hand side is not finite"):
        op.pcg(b, op.diagonal(), tol=1e-8)


def test_indefinite_operator_raises(ctx, form):
    """Negated geometric factors (make_operator rejects alpha < 0): p^T A p < 0
    on the first direction (pcg.cpp:76-82)."""
    pr = oracle.setup("bp5", 7, (2, 2, 2), "sine")
    pts, _ = oracle.quadrature("gll", pr.q)
    op = capi.Operator(ctx, p=pr.p, q=pr.q, m=1, num_elements=pr.num_elements, n_L=pr.num_nodes,
                       interp1d=pr.interp1d, grad1d=pr.grad1d, qpoints=pts, indices=pr.indices,
                       diff_qdata=-pr.qdata("diff"), alpha=1.0, beta=0.0,
                       constrained=pr.constrained)
    with pytest.raises(capi.HxfNumericError, match="indefinite direction"):
        op.pcg(pr.rhs, None, tol=1e-8)


def test_nan_in_operator_raises(ctx, form):
    pr = oracle.setup("bp5", 7, (2, 2, 2), "sine")
    pts, _ = oracle.quadrature("gll", pr.q)
    qd = pr.qdata("diff").copy()
    qd[100] = np.nan
    op = capi.Operator(ctx, p=pr.p, q=pr.q, m=1, num_elements=pr.num_elements, n_L=pr.num_nodes,
                       interp1d=pr.interp1d, grad1d=pr.grad1d, qpoints=pts, indices=pr.indices,
                       diff_qdata=qd, alpha=1.0, beta=0.0, constrained=pr.constrained)
    with pytest.raises(capi.HxfNumericError, match="NaN in operator apply"):
        op.pcg(pr.rhs, None, tol=1e-8)
