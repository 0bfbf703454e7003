"""B200-native BP1-BP6 matrix-free operator + Jacobi-PCG (drop-in for hexfem).

The compute path is hand-written CUDA for sm_100a behind the C-ABI of
``include/hxf.h`` (``_native/libhxf.so``); ``capi`` binds it directly.
"""
from . import capi  # noqa: F401

__all__ = ["capi"]
