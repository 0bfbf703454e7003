"""B200-native BP1-BP6 matrix-free operators + Jacobi-PCG — a drop-in for the
reference's (hexfem) operator path.

Python API (mirrors ``hexfem._core``, proj/bindings/module.cpp:78-213):
``quadrature``, ``basis``/``Basis``, ``setup`` -> ``Problem`` with
``apply/diagonal/assemble/solve/l2_error``, ``run_bench``.  Everything
operator-sized runs as hand-written sm_100a CUDA behind the C-ABI of
``include/hxf.h`` (``_native/libhxf.so``); ``capi`` binds that C-ABI directly.
There is no CPU fallback: importing without the built native library fails.
"""
from . import capi  # noqa: F401
from ._core import Basis, Problem, __version__, basis, quadrature, run_bench, setup  # noqa: F401

__all__ = ["Basis", "Problem", "__version__", "basis", "capi", "quadrature", "run_bench", "setup"]
