"""The C restatement vs the reference itself (oracle/_ref, compiled from
/root/reference/proj/src).  Skipped where oracle/_ref was not built."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.skipif(not oracle.available("reference"),
                                reason="oracle/_ref not built (make -C oracle ref)")

CASES = [
    ("bp1", 2, (3, 2, 2), "sine"), ("bp2", 3, (2, 2, 1), "none"), ("bp3", 3, (2, 3, 2), "sine"),
    ("bp4", 2, (2, 2, 2), "sine"), ("bp5", 5, (2, 2, 2), "sine"), ("bp6", 2, (3, 2, 2), "sine"),
    ("bp5", 9, (1, 2, 1), "sine"), ("bp3", 6, (2, 1, 1), "none"), ("bp5", 15, (1, 1, 1), "sine"),
]


@pytest.mark.parametrize("bp,p,dims,deform", CASES)
def test_restatement_bitwise_equals_reference(bp, p, dims, deform):
    a = oracle.setup(bp, p, dims, deform, impl="oracle")
    b = oracle.setup(bp, p, dims, deform, threads=4, impl="reference")
    assert np.array_equal(a.indices, b.indices)
    assert np.array_equal(a.rhs, b.rhs)
    x = oracle.seeded_uniform(a.size, 1234)
    assert np.array_equal(a.apply(x), b.apply(x))
    assert np.array_equal(a.diagonal(), b.diagonal())
    xa, ra = a.solve(tol=1e-9)
    xb, rb = b.solve(tol=1e-9)
    assert ra["iterations"] == rb["iterations"]
    assert np.array_equal(xa, xb)
