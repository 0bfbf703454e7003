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
