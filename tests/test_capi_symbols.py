"""The drop-in boundary without a GPU: libhxf.so loads, exports every symbol
include/hxf.h declares, and fails loudly (HXF_ECUDA, no CPU fallback) when no
device is present."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2109_04996_b200 import capi

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "hxf.h").read_text()
    return sorted(set(re.findall(r"\b(hxf_[a-z_0-9]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(capi.LIB_PATH))
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_abi_version_and_error_channel():
    lib = capi.lib()
    assert lib.hxf_abi_version() == 2
    assert isinstance(lib.hxf_last_error(), bytes)


def test_no_cpu_fallback_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(capi.HxfError) as ei:
        capi.Context(0)
    assert ei.value.code == capi.HXF_ECUDA
    assert "no CUDA device" in str(ei.value)


def test_python_api_fails_loudly_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2109_04996_b200 as hx

    # host-only setup tables work; anything operator-sized needs the device
    assert hx.quadrature("gll", 3)[0].tolist() == [-1.0, 0.0, 1.0]
    with pytest.raises(RuntimeError, match="no CUDA device"):
        hx.setup("bp5", degree=2, dims=(1, 1, 1))


def test_host_tables_match_oracle_bitwise():
    """The product's own C++ setup tables (quadrature, basis) equal the
    reference's bit for bit (tests/golden/tables.npz)."""
    import numpy as np

    import paper_2109_04996_b200 as hx

    t = dict(np.load(ROOT / "tests" / "golden" / "tables.npz"))
    for kind, qs in (("gauss", range(1, 18)), ("gll", range(2, 18))):
        for q in qs:
            pts, wts = hx.quadrature(kind, q)
            assert np.array_equal(pts, t[f"quad_{kind}_{q}_pts"])
            assert np.array_equal(wts, t[f"quad_{kind}_{q}_wts"])
    for p in range(1, 16):
        for kind, q in (("gauss", p + 2), ("gll", p + 1)):
            b = hx.basis(p, kind, q)
            assert np.array_equal(b.interp1d, t[f"basis_{kind}_{p}_B"])
            assert np.array_equal(b.grad1d, t[f"basis_{kind}_{p}_G"])


def test_flops_estimate_matches_reference_formula():
    """hxf_flops_estimate is host arithmetic (no device): the reference's
    known answers (test_contraction.cpp:122-129) and the oracle's closed form."""
    import oracle

    assert capi.flops_estimate(1, 1, 1, "interp") == 28
    assert capi.flops_estimate(1, 1, 1, "grad") == 84
    for p in range(1, 16):
        for q in (p + 1, p + 2):
            for m in (1, 3):
                for mode in ("interp", "grad"):
                    assert capi.flops_estimate(p, q, m, mode) == oracle.flops_estimate(p, q, m, mode)
    # per-apply counts recorded by the reference's acceptance run
    # (acceptance.cpp:393-404, test_output.txt:21): 8 elements x (B + B^T)
    assert 8 * 2 * capi.flops_estimate(3, 4, 1, "grad") == 73728   # BP5 p=3 2^3
    assert 8 * 2 * capi.flops_estimate(3, 5, 1, "grad") == 117120  # BP3 p=3 2^3
