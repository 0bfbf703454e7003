"""ctypes binding of the hxf C-ABI (include/hxf.h) — the drop-in boundary.

This is the exact surface a reference-side FFI would bind.
Arrays may be numpy (HXF_HOST) or CUDA tensors / raw device pointers
(HXF_DEVICE).  There is no CPU fallback: every compute call fails loudly with
:class:`HxfError` when the native library or the GPU is missing.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_native" / "libhxf.so"

HXF_OK, HXF_EINVAL, HXF_ENUMERIC, HXF_ECUDA, HXF_ENCCL, HXF_EUNSUPPORTED = range(6)
HXF_HOST, HXF_DEVICE = 0, 1

# Every symbol include/hxf.h declares (checked by tests/test_capi_symbols.py).
EXPORTS = (
    "hxf_last_error", "hxf_abi_version", "hxf_launch_count", "hxf_context_create",
    "hxf_context_destroy", "hxf_context_stream", "hxf_operator_create", "hxf_operator_destroy",
    "hxf_operator_size", "hxf_operator_is_structured", "hxf_operator_apply",
    "hxf_operator_diagonal", "hxf_restriction_apply", "hxf_restriction_multiplicity",
    "hxf_basis_apply", "hxf_qfunction_apply", "hxf_qdata_compute", "hxf_pcg",
    "hxf_malloc", "hxf_free", "hxf_memcpy", "hxf_synchronize",
    "hxf_comm_unique_id", "hxf_comm_create_nccl", "hxf_comm_wrap_nccl", "hxf_comm_group_create",
    "hxf_comm_group_destroy", "hxf_comm_create_group", "hxf_comm_destroy", "hxf_comm_rank",
    "hxf_comm_size", "hxf_comm_allreduce_sum", "hxf_operator_set_partition",
    "hxf_operator_halo_sum", "hxf_pcg_host_batch", "hxf_debug_set_grid_cap",
    "hxf_debug_step_timestamps", "hxf_debug_set_op_kernel",
    "hxf_elem_restriction_create", "hxf_elem_restriction_destroy",
    "hxf_elem_restriction_is_structured", "hxf_elem_restriction_apply",
    "hxf_elem_restriction_multiplicity", "hxf_elem_restriction_gather_scalar",
    "hxf_contract_batch", "hxf_apply_tensor_3d", "hxf_flops_estimate", "hxf_box_fields",
    "hxf_operator_set_constrained", "hxf_comm_p2p_alloc", "hxf_comm_create_p2p", "hxf_comm_p2p_free",
)


class HxfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class HxfInvalidArgument(HxfError, ValueError):
    """HXF_EINVAL — the reference's std::invalid_argument."""


class HxfNumericError(HxfError):
    """HXF_ENUMERIC — the reference's std::runtime_error."""


class PartitionDesc(C.Structure):
    _fields_ = [("neighbor", (C.c_int * 2) * 3)]


class OperatorDesc(C.Structure):
    _fields_ = [
        ("p", C.c_int), ("q", C.c_int), ("m", C.c_int),
        ("num_elements", C.c_int64), ("n_L", C.c_int64),
        ("interp1d", C.c_void_p), ("grad1d", C.c_void_p), ("qpoints", C.c_void_p),
        ("indices", C.c_void_p), ("dims", C.c_int * 3),
        ("mass_qdata", C.c_void_p), ("diff_qdata", C.c_void_p), ("qdata_space", C.c_int),
        ("alpha", C.c_double), ("beta", C.c_double),
        ("constrained", C.c_void_p), ("n_constrained", C.c_int64), ("block", C.c_int),
    ]


class PcgOptions(C.Structure):
    _fields_ = [("tol_rel", C.c_double), ("max_iter", C.c_int), ("fixed_iterations", C.c_int),
                ("time_apply", C.c_int)]


class SolveReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int), ("converged", C.c_int),
        ("residual_history", C.c_void_p), ("history_capacity", C.c_int),
        ("apply_time_seconds", C.c_double), ("total_time_seconds", C.c_double),
    ]


_lib = None


def lib() -> C.CDLL:
    """Load libhxf.so (build it first: ``python -c 'import __graft_entry__ as g; g.build()'``)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise HxfError(HXF_ECUDA, f"native library missing: {LIB_PATH} (run build())")
    L = C.CDLL(str(LIB_PATH))
    P, I, I64, D = C.c_void_p, C.c_int, C.c_int64, C.c_double
    L.hxf_last_error.restype = C.c_char_p
    L.hxf_launch_count.restype = I64
    L.hxf_context_create.argtypes = [I, P, C.POINTER(P)]
    L.hxf_context_destroy.argtypes = [P]
    L.hxf_context_stream.restype = P
    L.hxf_context_stream.argtypes = [P]
    L.hxf_operator_create.argtypes = [P, C.POINTER(OperatorDesc), C.POINTER(P)]
    L.hxf_operator_destroy.argtypes = [P]
    L.hxf_operator_size.restype = I64
    L.hxf_operator_size.argtypes = [P]
    L.hxf_operator_is_structured.argtypes = [P]
    L.hxf_operator_apply.argtypes = [P, P, P, I, P]
    L.hxf_operator_diagonal.argtypes = [P, P, I]
    L.hxf_restriction_apply.argtypes = [P, I, P, P, I]
    L.hxf_restriction_multiplicity.argtypes = [P, P, I]
    L.hxf_basis_apply.argtypes = [P, I, I, P, P, I, I, I64, P, P, I]
    L.hxf_qfunction_apply.argtypes = [P, I, P, I64, I, I64, I64, P, P, I]
    L.hxf_qdata_compute.argtypes = [P, I, I, P, P, P, I64, I64, P, P, P, I, P, I]
    L.hxf_pcg.argtypes = [P, P, P, C.POINTER(PcgOptions), P, I, C.POINTER(SolveReport)]
    L.hxf_comm_unique_id.argtypes = [P]
    L.hxf_comm_create_nccl.argtypes = [P, I, I, P, C.POINTER(P)]
    L.hxf_comm_wrap_nccl.argtypes = [P, P, C.POINTER(P)]
    L.hxf_comm_group_create.argtypes = [I, C.POINTER(P)]
    L.hxf_comm_group_destroy.argtypes = [P]
    L.hxf_comm_create_group.argtypes = [P, P, I, C.POINTER(P)]
    L.hxf_comm_destroy.argtypes = [P]
    L.hxf_comm_rank.argtypes = [P]
    L.hxf_comm_size.argtypes = [P]
    L.hxf_comm_allreduce_sum.argtypes = [P, P, I64, P]
    L.hxf_operator_set_partition.argtypes = [P, P, C.POINTER(PartitionDesc)]
    L.hxf_operator_halo_sum.argtypes = [P, P, I]
    L.hxf_pcg_host_batch.argtypes = [P, I, P, P, C.POINTER(PcgOptions), P, P]
    L.hxf_debug_set_grid_cap.argtypes = [I]
    L.hxf_debug_step_timestamps.argtypes = [I, C.c_void_p]
    L.hxf_debug_set_op_kernel.argtypes = [I]
    L.hxf_elem_restriction_create.argtypes = [P, I, I, I64, I64, P, P, C.POINTER(P)]
    L.hxf_elem_restriction_destroy.argtypes = [P]
    L.hxf_elem_restriction_is_structured.argtypes = [P]
    L.hxf_elem_restriction_apply.argtypes = [P, I, P, I64, P, I64, I]
    L.hxf_elem_restriction_multiplicity.argtypes = [P, P, I64, I]
    L.hxf_elem_restriction_gather_scalar.argtypes = [P, P, I64, P, I64, I]
    L.hxf_contract_batch.argtypes = [P, P, I64, I, I, I, P, I64, P, I64, P, I64, I, I,
                                     C.POINTER(C.c_uint64)]
    L.hxf_apply_tensor_3d.argtypes = [P, I, I, P, P, I, I, I, P, I64, P, I64, I]
    L.hxf_box_fields.argtypes = [P, P, P, P, I, P, I, I, I, P, P, P, I]
    L.hxf_operator_set_constrained.argtypes = [P, P, D, I]
    L.hxf_comm_p2p_alloc.argtypes = [P, I, I64, C.POINTER(P), P]
    L.hxf_comm_create_p2p.argtypes = [P, I, I, I64, P, P, C.POINTER(P)]
    L.hxf_comm_p2p_free.argtypes = [P, P]
    L.hxf_flops_estimate.restype = C.c_uint64
    L.hxf_flops_estimate.argtypes = [I, I, I, I]
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == HXF_OK:
        return
    msg = lib().hxf_last_error().decode()
    if rc == HXF_EINVAL:
        raise HxfInvalidArgument(rc, msg)
    if rc == HXF_ENUMERIC:
        raise HxfNumericError(rc, msg)
    raise HxfError(rc, msg)


def set_op_kernel(choice: int) -> int:
    """Test knob (hxf_debug_set_op_kernel): 0 tuned dispatch, 1 line / pencil
    kernels instead of the tensor-core ones, 2 the general kernel; returns the
    previous choice."""
    return int(lib().hxf_debug_set_op_kernel(int(choice)))


def launch_count() -> int:
    return int(lib().hxf_launch_count())


def set_grid_cap(cap: int) -> int:
    """Cap the operator / PCG vector kernel grids (test knob; 0 = none).  Returns the old cap."""
    return int(lib().hxf_debug_set_grid_cap(int(cap)))


def flops_estimate(p: int, q: int, m: int, mode: str) -> int:
    """flops_estimate (contraction.cpp:334-340); mode 'interp' | 'grad'."""
    return int(lib().hxf_flops_estimate(p, q, m, 1 if mode == "grad" else 0))


def _empty_like_space(ref, n):
    if isinstance(ref, np.ndarray):
        return np.zeros(n)
    import torch
    return torch.empty(n, dtype=torch.float64, device=ref.device)


def _len(a) -> int:
    return 0 if a is None else int(a.size if isinstance(a, np.ndarray) else a.numel())


def _ptr(a):
    """(pointer, memspace) of a numpy array or a CUDA tensor."""
    if a is None:
        return None, HXF_HOST
    if isinstance(a, np.ndarray):
        assert a.flags["C_CONTIGUOUS"]
        return a.ctypes.data, HXF_HOST
    if hasattr(a, "data_ptr"):  # torch tensor
        assert a.is_contiguous()
        return a.data_ptr(), (HXF_DEVICE if a.is_cuda else HXF_HOST)
    raise TypeError(type(a))


def _f64(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float64)
    return a


class Context:
    def __init__(self, device: int = 0, nccl_comm=None):
        self._h = C.c_void_p()
        check(lib().hxf_context_create(device, nccl_comm, C.byref(self._h)))

    @property
    def handle(self):
        return self._h

    @property
    def stream(self) -> int:
        return lib().hxf_context_stream(self._h)

    def close(self):
        if self._h:
            lib().hxf_context_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- API-surface kernels ----
    def basis_apply(self, p, q, interp1d, grad1d, mode, direction, ne, u):
        """apply_basis_batch: mode 'interp'|'grad', direction 'forward'|'transpose'."""
        B = np.ascontiguousarray(interp1d, dtype=np.float64)
        G = np.ascontiguousarray(grad1d, dtype=np.float64)
        grad = mode == "grad"
        tr = direction == "transpose"
        nd3, nq3 = (p + 1) ** 3, q ** 3
        out_e = 3 * nq3 if (grad and not tr) else (nq3 if not tr else nd3)
        u = _f64(u)
        up, space = _ptr(u)
        if space == HXF_HOST:
            out = np.zeros(ne * out_e)
        else:
            import torch
            out = torch.empty(ne * out_e, dtype=torch.float64, device=u.device)
        op_, _ = _ptr(out)
        check(lib().hxf_basis_apply(self._h, p, q, B.ctypes.data, G.ctypes.data, int(grad), int(tr),
                                    ne, up, op_, space))
        return out

    def qfunction_apply(self, kind, qdata, num_elements, nq, e0, ne, u):
        qd = _f64(qdata)
        u = _f64(u)
        qp, space = _ptr(qd)
        up, _ = _ptr(u)
        k = 0 if kind == "mass" else 1
        n = (1 if k == 0 else 3) * ne * nq
        if space == HXF_HOST:
            out = np.zeros(n)
        else:
            import torch
            out = torch.empty(n, dtype=torch.float64, device=u.device)
        op_, _ = _ptr(out)
        check(lib().hxf_qfunction_apply(self._h, k, qp, num_elements, nq, e0, ne, up, op_, space))
        return out

    def qdata_compute(self, p, q, interp1d, grad1d, qweights, num_elements, n_L, coords,
                      indices=None, dims=None, kind="diffusion"):
        B = np.ascontiguousarray(interp1d, dtype=np.float64)
        G = np.ascontiguousarray(grad1d, dtype=np.float64)
        w = np.ascontiguousarray(qweights, dtype=np.float64)
        coords = _f64(coords)
        cp, space = _ptr(coords)
        idx = None if indices is None else np.ascontiguousarray(indices, dtype=np.int64)
        dims_arr = (C.c_int * 3)(*(dims if dims is not None else (0, 0, 0)))
        K = 1 if kind == "mass" else 6
        n = num_elements * K * q ** 3
        if space == HXF_HOST:
            out = np.zeros(n)
        else:
            import torch
            out = torch.empty(n, dtype=torch.float64, device=coords.device)
        op_, _ = _ptr(out)
        check(lib().hxf_qdata_compute(self._h, p, q, B.ctypes.data, G.ctypes.data, w.ctypes.data,
                                      num_elements, n_L, cp,
                                      None if idx is None else idx.ctypes.data, dims_arr,
                                      0 if kind == "mass" else 1, op_, space))
        return out


    def contract_batch(self, matrix, n_out, n_in, dim, in_shape, ne, u, out=None,
                       accumulate=False, flops=None):
        """contract_batch (contraction.cpp:177-206).  `flops`: a one-element list
        used as the FlopCounter (incremented by 2 per multiply-add)."""
        M = np.ascontiguousarray(matrix, dtype=np.float64).reshape(-1)
        u = _f64(u)
        up, space = _ptr(u)
        in_elem = int(in_shape[0]) * int(in_shape[1]) * int(in_shape[2])
        out_n = ne * (in_elem // max(n_in, 1)) * n_out if n_in > 0 else 0
        if out is None:
            out = _empty_like_space(u, out_n)
            if accumulate:
                raise ValueError("contract_batch: accumulate needs an output array")
        out = _f64(out)
        shape = (C.c_int * 3)(*[int(v) for v in in_shape])
        cnt = C.c_uint64(0 if flops is None else int(flops[0]))
        check(lib().hxf_contract_batch(self._h, M.ctypes.data, M.size, n_out, n_in, dim, shape, ne,
                                       up, _len(u), _ptr(out)[0], _len(out), int(bool(accumulate)),
                                       space, C.byref(cnt)))
        if flops is not None:
            flops[0] = cnt.value
        return out

    def apply_tensor_3d(self, p, q, interp1d, grad1d, mode, direction, m, u):
        """apply_tensor_3d (tensor_basis.cpp:73-99): one element, m components."""
        B = np.ascontiguousarray(interp1d, dtype=np.float64)
        G = np.ascontiguousarray(grad1d, dtype=np.float64)
        grad, tr = mode == "grad", direction == "transpose"
        nd3, nq3 = (p + 1) ** 3, q ** 3
        out_e = nd3 if tr else (3 * nq3 if grad else nq3)
        u = _f64(u)
        up, space = _ptr(u)
        out = _empty_like_space(u, m * out_e)
        check(lib().hxf_apply_tensor_3d(self._h, p, q, B.ctypes.data, G.ctypes.data, int(grad),
                                        int(tr), m, up, _len(u), _ptr(out)[0], _len(out), space))
        return out


class ElemRestriction:
    """hxf_elem_restriction_* — the reference's ElemRestriction (restriction.hpp:14-50)."""

    def __init__(self, ctx: Context, *, p, m, num_elements, n_L, indices=None, dims=None):
        self.ctx = ctx
        idx = None if indices is None else np.ascontiguousarray(indices, dtype=np.int64)
        dims_arr = (C.c_int * 3)(*(dims if dims is not None else (0, 0, 0)))
        self._h = C.c_void_p()
        check(lib().hxf_elem_restriction_create(ctx.handle, p, m, num_elements, n_L,
                                                None if idx is None else idx.ctypes.data,
                                                dims_arr, C.byref(self._h)))
        self.p, self.m, self.num_elements, self.n_L = p, m, num_elements, n_L
        self.elem_size = (p + 1) ** 3

    @property
    def structured(self) -> bool:
        return bool(lib().hxf_elem_restriction_is_structured(self._h))

    def close(self):
        if self._h:
            lib().hxf_elem_restriction_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run(self, fn, v, n_out, *extra):
        v = _f64(v)
        vp, space = _ptr(v)
        out = _empty_like_space(v, n_out)
        check(fn(self._h, *extra, vp, _len(v), _ptr(out)[0], _len(out), space))
        return out

    def apply_g(self, l_vec):
        return self._run(lib().hxf_elem_restriction_apply, l_vec,
                         self.m * self.num_elements * self.elem_size, 0)

    def apply_g_transpose(self, e_vec):
        return self._run(lib().hxf_elem_restriction_apply, e_vec, self.m * self.n_L, 1)

    def gather_scalar(self, e_scalar):
        return self._run(lib().hxf_elem_restriction_gather_scalar, e_scalar, self.n_L)

    def multiplicity(self):
        out = np.zeros(self.n_L)
        check(lib().hxf_elem_restriction_multiplicity(self._h, out.ctypes.data, out.size, HXF_HOST))
        return out


class Operator:
    """hxf_operator_create over reference-shaped arrays (make_operator's inputs)."""

    def __init__(self, ctx: Context, *, p, q, m, num_elements, n_L, interp1d, grad1d,
                 qpoints=None, indices=None, dims=None, mass_qdata=None, diff_qdata=None,
                 alpha=0.0, beta=0.0, constrained=None):
        self.ctx = ctx
        keep = []

        def hold(a, dtype=np.float64):
            if a is None:
                return None
            if isinstance(a, np.ndarray) or isinstance(a, (list, tuple)):
                a = np.ascontiguousarray(a, dtype=dtype)
            keep.append(a)
            return _ptr(a)[0]

        d = OperatorDesc()
        d.p, d.q, d.m = p, q, m
        d.num_elements, d.n_L = num_elements, n_L
        d.interp1d = hold(interp1d)
        d.grad1d = hold(grad1d)
        d.qpoints = hold(qpoints)
        d.indices = hold(indices, np.int64)
        d.dims = (C.c_int * 3)(*(dims if dims is not None else (0, 0, 0)))
        qd_any = diff_qdata if diff_qdata is not None else mass_qdata
        d.qdata_space = _ptr(_f64(qd_any))[1] if qd_any is not None else HXF_HOST
        d.mass_qdata = hold(_f64(mass_qdata))
        d.diff_qdata = hold(_f64(diff_qdata))
        d.alpha, d.beta = float(alpha), float(beta)
        cons = None if constrained is None else np.ascontiguousarray(constrained, dtype=np.int64)
        d.constrained = hold(cons, np.int64)
        d.n_constrained = 0 if cons is None else int(cons.size)
        d.block = 8
        self._h = C.c_void_p()
        check(lib().hxf_operator_create(ctx.handle, C.byref(d), C.byref(self._h)))
        self.size = int(lib().hxf_operator_size(self._h))
        self.m, self.n_L, self.num_elements = m, n_L, num_elements
        self.elem_size = (p + 1) ** 3

    @property
    def structured(self) -> bool:
        return bool(lib().hxf_operator_is_structured(self._h))

    def close(self):
        if self._h:
            lib().hxf_operator_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _out_like(self, x, n):
        if isinstance(x, np.ndarray):
            return np.zeros(n)
        import torch
        return torch.empty(n, dtype=torch.float64, device=x.device)

    def apply(self, x, y=None, stream=None):
        x = _f64(x)
        xp, space = _ptr(x)
        if y is None:
            y = self._out_like(x, self.size)
        yp, _ = _ptr(y)
        check(lib().hxf_operator_apply(self._h, xp, yp, space, stream))
        return y

    def diagonal(self, device=None):
        if device is None:
            d = np.zeros(self.size)
        else:
            import torch
            d = torch.empty(self.size, dtype=torch.float64, device=device)
        dp, space = _ptr(d)
        check(lib().hxf_operator_diagonal(self._h, dp, space))
        return d

    def restriction(self, v, transpose=False):
        v = _f64(v)
        n = self.m * self.n_L if transpose else self.m * self.num_elements * self.elem_size
        out = self._out_like(v, n)
        vp, space = _ptr(v)
        check(lib().hxf_restriction_apply(self._h, int(transpose), vp, _ptr(out)[0], space))
        return out

    def multiplicity(self):
        out = np.zeros(self.n_L)
        check(lib().hxf_restriction_multiplicity(self._h, out.ctypes.data, HXF_HOST))
        return out

    def pcg(self, b, diag=None, tol=1e-8, max_iter=2000, fixed_iterations=None, x=None,
            time_apply=True):
        b = _f64(b)
        diag = _f64(diag)
        bp, space = _ptr(b)
        if x is None:
            x = self._out_like(b, self.size)
        opts = PcgOptions(tol, max_iter, -1 if fixed_iterations is None else fixed_iterations,
                          int(bool(time_apply)))
        cap = (fixed_iterations if fixed_iterations is not None else max_iter) + 2
        hist = np.zeros(cap)
        rep = SolveReport(0, 0, hist.ctypes.data, cap, 0.0, 0.0)
        check(lib().hxf_pcg(self._h, bp, _ptr(diag)[0], C.byref(opts), _ptr(x)[0], space,
                            C.byref(rep)))
        report = {
            "iterations": rep.iterations, "converged": bool(rep.converged),
            "residual_history": hist[: rep.iterations + 1].copy(),
            "apply_time_seconds": rep.apply_time_seconds,
            "total_time_seconds": rep.total_time_seconds,
        }
        return x, report


# ---- partitioned box (include/hxf.h "partitioned box") ----------------------
COMM_ID_BYTES = 128


def comm_unique_id() -> bytes:
    buf = (C.c_ubyte * COMM_ID_BYTES)()
    check(lib().hxf_comm_unique_id(buf))
    return bytes(buf)


class CommGroup:
    """In-process group: n sub-domains, one host thread each (ctypes drops the GIL)."""

    def __init__(self, nranks: int):
        self._h = C.c_void_p()
        check(lib().hxf_comm_group_create(nranks, C.byref(self._h)))
        self.size = nranks

    def close(self):
        if self._h:
            lib().hxf_comm_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    def __init__(self, ctx: Context, *, group: CommGroup = None, rank: int = 0,
                 nranks: int = 1, unique_id: bytes = None):
        self.ctx = ctx
        self._h = C.c_void_p()
        if group is not None:
            check(lib().hxf_comm_create_group(ctx.handle, group._h, rank, C.byref(self._h)))
        else:
            buf = (C.c_ubyte * COMM_ID_BYTES).from_buffer_copy(unique_id)
            check(lib().hxf_comm_create_nccl(ctx.handle, nranks, rank, buf, C.byref(self._h)))

    @property
    def rank(self) -> int:
        return int(lib().hxf_comm_rank(self._h))

    @property
    def size(self) -> int:
        return int(lib().hxf_comm_size(self._h))

    def allreduce_sum(self, t) -> None:
        """In-place sum of a CUDA float64 tensor across ranks."""
        check(lib().hxf_comm_allreduce_sum(self._h, t.data_ptr(), t.numel(), None))

    def close(self):
        if self._h:
            lib().hxf_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def set_partition(op: Operator, comm: Comm, neighbor) -> None:
    """neighbor[axis][side] = rank sharing the low (0) / high (1) face plane, -1 = none."""
    d = PartitionDesc()
    for a in range(3):
        for s in range(2):
            d.neighbor[a][s] = int(neighbor[a][s])
    check(lib().hxf_operator_set_partition(op._h, comm._h, C.byref(d)))
    op._comm = comm  # keep the communicator alive with the operator


def halo_sum(op: Operator, v):
    v = _f64(v)
    vp, space = _ptr(v)
    check(lib().hxf_operator_halo_sum(op._h, vp, space))
    return v
