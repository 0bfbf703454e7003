"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the BP operator + PCG path.

Never imported by the product package (``paper_2109_04996_b200``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may use it, and only as the checker.

Two interchangeable implementations behind the same ``orc_*`` C entry points:

* ``impl="oracle"`` — ``liboracle.so``, our plain-C restatement of the
  reference algorithm (``hexfem_oracle.c``), built by ``make -C oracle``;
* ``impl="reference"`` — ``_ref/libref_capi.so``, a flat C shim over the
  UNMODIFIED reference library compiled from ``/root/reference/proj/src``
  (built here only; the built ``.so`` travels to the GPU box).

Parity of the restatement is pinned by ``tests/test_oracle_ref.py`` (bitwise
against the reference) and ``tests/test_oracle_golden.py`` (golden vectors and
the reference's own known-answer tests).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
_LIBS: dict[str, C.CDLL] = {}

BP_IDS = {f"bp{i}": i for i in range(1, 7)}


def lib_path(impl: str = "oracle") -> Path:
    if impl == "oracle":
        return HERE / "liboracle.so"
    if impl == "reference":
        return HERE / "_ref" / "libref_capi.so"
    raise ValueError(impl)


def available(impl: str = "oracle") -> bool:
    return lib_path(impl).exists()


def build(impl: str = "oracle") -> None:
    import subprocess

    target = "oracle" if impl == "oracle" else "ref"
    subprocess.run(["make", "-s", "-C", str(HERE), target], check=True)


def _lib(impl: str) -> C.CDLL:
    if impl in _LIBS:
        return _LIBS[impl]
    path = lib_path(impl)
    if not path.exists():
        if impl == "oracle":
            build("oracle")
        else:
            raise FileNotFoundError(f"{path} not built (make -C oracle ref)")
    L = C.CDLL(str(path))
    P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
    pd, pi64, pi = C.POINTER(C.c_double), C.POINTER(C.c_int64), C.POINTER(C.c_int)
    L.orc_last_error.restype = C.c_char_p
    L.orc_impl_name.restype = C.c_char_p
    L.orc_setup.restype = P
    L.orc_setup.argtypes = [I, I, I, I, I, I, I]
    L.orc_free.argtypes = [P]
    L.orc_info.argtypes = [P, pi64]
    for name in ("orc_rhs", "orc_exact", "orc_coords", "orc_interp1d", "orc_grad1d"):
        getattr(L, name).restype = pd
        getattr(L, name).argtypes = [P]
    for name in ("orc_indices", "orc_constrained"):
        getattr(L, name).restype = pi64
        getattr(L, name).argtypes = [P]
    L.orc_qdata.restype = pd
    L.orc_qdata.argtypes = [P, I]
    L.orc_alpha.restype = D
    L.orc_alpha.argtypes = [P]
    L.orc_beta.restype = D
    L.orc_beta.argtypes = [P]
    L.orc_apply.argtypes = [P, pd, pd]
    L.orc_diagonal.argtypes = [P, pd]
    L.orc_solve.argtypes = [P, D, I, I, I, pd, pd, I, pi, pi]
    L.orc_l2_error.restype = D
    L.orc_l2_error.argtypes = [P, pd]
    L.orc_quadrature.argtypes = [I, I, pd, pd]
    L.orc_basis.argtypes = [I, I, I, pd, pd]
    L.orc_apply_basis.argtypes = [I, I, I, I, I, I64, pd, I64, pd, I64]
    U64 = C.c_uint64
    L.orc_contract_batch.argtypes = [pd, I64, I, I, I, pi, I64, pd, I64, pd, I64, I,
                                     C.POINTER(U64)]
    L.orc_apply_tensor_3d.argtypes = [I, I, I, I, I, I, pd, I64, pd, I64]
    L.orc_flops_estimate.restype = U64
    L.orc_flops_estimate.argtypes = [I, I, I, I]
    L.orc_apply_basis_counted.argtypes = [I, I, I, I, I, I64, pd, I64, pd, I64, C.POINTER(U64)]
    L.orc_gather_scalar.argtypes = [P, pd, I64, pd, I64]
    if impl == "reference":
        L.orc_run_bench.argtypes = [I, I, I, I, I, I, I, I, pd]
        L.orc_sweep_model.argtypes = [I, I, pi, I, pi, I, I, D, D, C.c_char_p, I64, pd]
        L.orc_record_json.argtypes = [C.c_char_p, I, I, I64, I64, I, I, D, D, D, C.c_char_p, I64]
    _LIBS[impl] = L
    return L


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _check(L, rc: int) -> None:
    if rc != 0:
        msg = L.orc_last_error().decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)


def _kind(kind: str) -> int:
    if kind in ("gauss", "gauss-legendre"):
        return 0
    if kind in ("gll", "gauss-lobatto", "gauss-lobatto-legendre"):
        return 1
    raise ValueError(f"unknown quadrature kind: {kind}")


def quadrature(kind: str, q: int, impl: str = "oracle"):
    L = _lib(impl)
    pts, wts = np.zeros(q), np.zeros(q)
    _check(L, L.orc_quadrature(_kind(kind), q, _dp(pts), _dp(wts)))
    return pts, wts


def basis(p: int, kind: str, q: int, impl: str = "oracle"):
    L = _lib(impl)
    B, G = np.zeros((q, p + 1)), np.zeros((q, p + 1))
    _check(L, L.orc_basis(p, _kind(kind), q, _dp(B), _dp(G)))
    return B, G


def apply_basis(p: int, kind: str, q: int, mode: str, direction: str, ne: int,
                u: np.ndarray, impl: str = "oracle") -> np.ndarray:
    """apply_basis_batch (src/contraction.cpp:248-332); grad layout (d*ne+e)*q^3."""
    L = _lib(impl)
    grad = mode == "grad"
    tr = direction == "transpose"
    nd3, nq3 = (p + 1) ** 3, q ** 3
    out_e = 3 * nq3 if (grad and not tr) else (nq3 if not tr else nd3)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(ne * out_e)
    _check(L, L.orc_apply_basis(p, _kind(kind), q, int(grad), int(tr), ne, _dp(u), u.size,
                                _dp(out), out.size))
    return out


def contract_batch(matrix, n_out: int, n_in: int, dim: int, shape, ne: int, u,
                   out=None, accumulate: bool = False, impl: str = "oracle"):
    """contract_batch (src/contraction.cpp:177-206) -> (out, flops counted)."""
    L = _lib(impl)
    M = np.ascontiguousarray(matrix, dtype=np.float64).reshape(-1)
    u = np.ascontiguousarray(u, dtype=np.float64)
    in_elem = int(shape[0]) * int(shape[1]) * int(shape[2])
    n = ne * (in_elem // max(n_in, 1)) * n_out if n_in > 0 else 0
    out = np.zeros(n) if out is None else np.array(out, dtype=np.float64, copy=True)
    sh = np.ascontiguousarray(shape, dtype=np.int32)
    cnt = C.c_uint64(0)
    _check(L, L.orc_contract_batch(_dp(M), M.size, n_out, n_in, dim,
                                   sh.ctypes.data_as(C.POINTER(C.c_int)), ne, _dp(u), u.size,
                                   _dp(out), out.size, int(bool(accumulate)), C.byref(cnt)))
    return out, int(cnt.value)


def apply_tensor_3d(p: int, kind: str, q: int, mode: str, direction: str, m: int, u,
                    impl: str = "oracle") -> np.ndarray:
    """apply_tensor_3d (src/tensor_basis.cpp:73-99)."""
    L = _lib(impl)
    grad, tr = mode == "grad", direction == "transpose"
    nd3, nq3 = (p + 1) ** 3, q ** 3
    out_e = nd3 if tr else (3 * nq3 if grad else nq3)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(m * out_e)
    _check(L, L.orc_apply_tensor_3d(p, _kind(kind), q, int(grad), int(tr), m, _dp(u), u.size,
                                    _dp(out), out.size))
    return out


def flops_estimate(p: int, q: int, m: int, mode: str, impl: str = "oracle") -> int:
    """flops_estimate (src/contraction.cpp:334-340)."""
    return int(_lib(impl).orc_flops_estimate(p, q, m, 1 if mode == "grad" else 0))


def apply_basis_counted(p: int, kind: str, q: int, mode: str, direction: str, ne: int, u,
                        impl: str = "oracle"):
    """apply_basis_batch with a FlopCounter attached -> (out, counted flops)."""
    L = _lib(impl)
    grad, tr = mode == "grad", direction == "transpose"
    nd3, nq3 = (p + 1) ** 3, q ** 3
    out_e = 3 * nq3 if (grad and not tr) else (nq3 if not tr else nd3)
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros(ne * out_e)
    cnt = C.c_uint64(0)
    _check(L, L.orc_apply_basis_counted(p, _kind(kind), q, int(grad), int(tr), ne, _dp(u), u.size,
                                        _dp(out), out.size, C.byref(cnt)))
    return out, int(cnt.value)


class Problem:
    """One BP problem built by the oracle's bp_setup (src/bench.cpp:64-119)."""

    def __init__(self, bp: str, degree: int, dims, deform: str = "none", threads: int = 1,
                 impl: str = "oracle"):
        self.impl = impl
        self._L = _lib(impl)
        self.bp = bp
        dims = tuple(int(d) for d in dims)
        h = self._L.orc_setup(BP_IDS[bp], degree, dims[0], dims[1], dims[2],
                              1 if deform == "sine" else 0, threads)
        if not h:
            raise ValueError(self._L.orc_last_error().decode())
        self._h = C.c_void_p(h)
        info = np.zeros(10, dtype=np.int64)
        self._L.orc_info(self._h, info.ctypes.data_as(C.POINTER(C.c_int64)))
        (self.components, self.num_nodes, self.num_elements, self.elem_size, self.nq, self.q,
         self.n, self.n_constrained, self.p, self.nodes_x) = (int(v) for v in info)
        self.dims = dims
        self.deform = deform
        self.size = self.components * self.num_nodes

    def __del__(self):
        try:
            self._L.orc_free(self._h)
        except Exception:
            pass

    def _arr(self, ptr, n, dtype=np.float64) -> np.ndarray:
        if not ptr or n == 0:
            return None if not ptr else np.zeros(0, dtype=dtype)
        return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)

    @property
    def rhs(self):
        return self._arr(self._L.orc_rhs(self._h), self.size)

    @property
    def exact(self):
        return self._arr(self._L.orc_exact(self._h), self.size)

    @property
    def coords(self):
        return self._arr(self._L.orc_coords(self._h), 3 * self.num_nodes)

    @property
    def indices(self):
        return self._arr(self._L.orc_indices(self._h), self.num_elements * self.elem_size,
                         np.int64)

    @property
    def constrained(self):
        if self.n_constrained == 0:
            return np.zeros(0, dtype=np.int64)
        return self._arr(self._L.orc_constrained(self._h), self.n_constrained, np.int64)

    def qdata(self, kind: str):
        k = 0 if kind == "mass" else 1
        n = self.num_elements * self.nq * (1 if k == 0 else 6)
        ptr = self._L.orc_qdata(self._h, k)
        return self._arr(ptr, n) if ptr else None

    @property
    def interp1d(self):
        return self._arr(self._L.orc_interp1d(self._h), self.q * (self.p + 1)).reshape(
            self.q, self.p + 1)

    @property
    def grad1d(self):
        return self._arr(self._L.orc_grad1d(self._h), self.q * (self.p + 1)).reshape(
            self.q, self.p + 1)

    @property
    def alpha(self):
        return self._L.orc_alpha(self._h)

    @property
    def beta(self):
        return self._L.orc_beta(self._h)

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        assert x.size == self.size
        y = np.zeros(self.size)
        _check(self._L, self._L.orc_apply(self._h, _dp(x), _dp(y)))
        return y

    def diagonal(self) -> np.ndarray:
        d = np.zeros(self.size)
        _check(self._L, self._L.orc_diagonal(self._h, _dp(d)))
        return d

    def solve(self, tol=1e-8, max_iter=2000, jacobi=True, fixed_iterations=None):
        x = np.zeros(self.size)
        cap = (fixed_iterations if fixed_iterations is not None else max_iter) + 2
        hist = np.zeros(cap)
        it, conv = C.c_int(0), C.c_int(0)
        _check(self._L, self._L.orc_solve(self._h, tol, max_iter, int(bool(jacobi)),
                                          -1 if fixed_iterations is None else fixed_iterations,
                                          _dp(x), _dp(hist), cap, C.byref(it), C.byref(conv)))
        report = {"iterations": it.value, "converged": bool(conv.value),
                  "residual_history": hist[: it.value + 1].copy()}
        return x, report

    def gather_scalar(self, e_scalar: np.ndarray) -> np.ndarray:
        """gather_scalar (src/restriction.cpp:86-106) over this problem's restriction."""
        e = np.ascontiguousarray(e_scalar, dtype=np.float64)
        out = np.zeros(self.num_nodes)
        _check(self._L, self._L.orc_gather_scalar(self._h, _dp(e), e.size, _dp(out), out.size))
        return out

    def l2_error(self, u: np.ndarray) -> float:
        u = np.ascontiguousarray(u, dtype=np.float64)
        return self._L.orc_l2_error(self._h, _dp(u))


def setup(bp: str, degree: int, dims, deform: str = "none", threads: int = 1,
          impl: str = "oracle") -> Problem:
    return Problem(bp, degree, dims, deform, threads, impl)


def run_bench_reference(bp: str, degree: int, dims, threads: int, iters: int,
                        deform: str = "none") -> dict:
    """The reference's own run_bench (src/bench.cpp:191-229), via oracle/_ref."""
    L = _lib("reference")
    rec = np.zeros(6)
    dims = tuple(int(d) for d in dims)
    _check(L, L.orc_run_bench(BP_IDS[bp], degree, dims[0], dims[1], dims[2],
                              1 if deform == "sine" else 0, threads, iters, _dp(rec)))
    return {"n": int(rec[0]), "iterations": int(rec[1]), "seconds": rec[2], "E": int(rec[3]),
            "q": int(rec[4]), "dofs_rate": rec[5], "P": threads}


def seeded_uniform(n: int, seed: int) -> np.ndarray:
    """U(-1,1) test vector (numpy PCG64; both sides of every comparison get the same one)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def rel_max_diff(a, b) -> float:
    """max|a-b| / max|a| — the reference's relative error (tests/oracle_helpers.hpp:74-81)."""
    a = np.asarray(a)
    b = np.asarray(b)
    scale = float(np.max(np.abs(a))) if a.size else 0.0
    diff = float(np.max(np.abs(a - b))) if a.size else 0.0
    return diff / scale if scale > 0 else diff


class RefWithBackend:
    """A reference BpProblem (oracle/_ref) driven both by the reference (CPU)
    and by the reference-side integration integration/hexfem_hxf.cpp (GPU).
    which = 0 reference, 1 hxf backend."""

    def __init__(self, bp: str, degree: int, dims, deform: str = "none", threads: int = 2):
        path = HERE / "_ref" / "libref_hxf.so"
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle ref after the product)")
        L = C.CDLL(str(path))
        P, I, D = C.c_void_p, C.c_int, C.c_double
        pd, pi = C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.orh_last_error.restype = C.c_char_p
        L.orh_setup.restype = P
        L.orh_setup.argtypes = [I, I, I, I, I, I, I]
        L.orh_free.argtypes = [P]
        L.orh_size.restype = C.c_int64
        L.orh_size.argtypes = [P]
        L.orh_apply.argtypes = [P, I, pd, pd]
        L.orh_diagonal.argtypes = [P, I, pd]
        L.orh_solve.argtypes = [P, I, D, I, pd, pi, pi]
        U64p = C.POINTER(C.c_uint64)
        I64 = C.c_int64
        L.orh_scale_qdata.argtypes = [P, D]
        L.orh_apply_counted.argtypes = [P, I, pd, pd, U64p]
        L.orh_restriction.argtypes = [P, I, I, pd, I64, pd, I64]
        L.orh_basis.argtypes = [P, I, I, I, I, I64, pd, I64, pd, I64, U64p]
        L.orh_contract.argtypes = [I, pd, I64, I, I, I, C.POINTER(C.c_int), I64, pd, I64, pd, I64,
                                   I, U64p]
        L.orh_flops_estimate.restype = C.c_uint64
        L.orh_flops_estimate.argtypes = [I, I, I, I, I]
        self._L = L
        dims = tuple(int(d) for d in dims)
        h = L.orh_setup(BP_IDS[bp], degree, dims[0], dims[1], dims[2],
                        1 if deform == "sine" else 0, threads)
        if not h:
            raise ValueError(L.orh_last_error().decode())
        self._h = C.c_void_p(h)
        self.size = int(L.orh_size(self._h))

    def _ck(self, rc):
        if rc:
            raise (ValueError if rc == 1 else RuntimeError)(self._L.orh_last_error().decode())

    def apply(self, x, which):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.size)
        self._ck(self._L.orh_apply(self._h, which, _dp(x), _dp(y)))
        return y

    def diagonal(self, which):
        d = np.zeros(self.size)
        self._ck(self._L.orh_diagonal(self._h, which, _dp(d)))
        return d

    def scale_qdata(self, s: float) -> None:
        """Scale the reference operator's qdata in place (same addresses)."""
        self._L.orh_scale_qdata(self._h, float(s))

    def apply_counted(self, x, which):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.size)
        cnt = C.c_uint64(0)
        self._ck(self._L.orh_apply_counted(self._h, which, _dp(x), _dp(y), C.byref(cnt)))
        return y, int(cnt.value)

    def restriction(self, which, what, v, n_out):
        """what: 'apply_g' | 'apply_g_transpose' | 'gather_scalar' | 'multiplicity'."""
        code = ["apply_g", "apply_g_transpose", "gather_scalar", "multiplicity"].index(what)
        v = np.ascontiguousarray(v if v is not None else np.zeros(0), dtype=np.float64)
        out = np.zeros(n_out)
        self._ck(self._L.orh_restriction(self._h, which, code, _dp(v), v.size, _dp(out), out.size))
        return out

    def basis(self, which, what, mode, direction, ne_or_m, v, n_out):
        """what: 'batch' (apply_basis_batch, ne blocks) | 'tensor3d' (m components)."""
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros(n_out)
        cnt = C.c_uint64(0)
        self._ck(self._L.orh_basis(self._h, which, 0 if what == "batch" else 1,
                                   int(mode == "grad"), int(direction == "transpose"), ne_or_m,
                                   _dp(v), v.size, _dp(out), out.size, C.byref(cnt)))
        return out, int(cnt.value)

    def contract(self, which, M, n_out, n_in, dim, shape, ne, u, out, accumulate):
        M = np.ascontiguousarray(M, dtype=np.float64)
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = np.array(out, dtype=np.float64, copy=True)
        sh = (C.c_int * 3)(*shape)
        cnt = C.c_uint64(0)
        self._ck(self._L.orh_contract(which, _dp(M), M.size, n_out, n_in, dim, sh, ne, _dp(u),
                                      u.size, _dp(out), out.size, int(accumulate), C.byref(cnt)))
        return out, int(cnt.value)

    def flops_estimate(self, which, p, q, m, mode):
        return int(self._L.orh_flops_estimate(which, p, q, m, int(mode == "grad")))

    def solve(self, which, tol=1e-8, jacobi=True):
        x = np.zeros(self.size)
        it, conv = C.c_int(0), C.c_int(0)
        self._ck(self._L.orh_solve(self._h, which, tol, int(jacobi), _dp(x), C.byref(it),
                                   C.byref(conv)))
        return x, it.value, bool(conv.value)

    def __del__(self):
        try:
            self._L.orh_free(self._h)
        except Exception:
            pass


def sweep_model_reference(bp: str, p: int, dims_list, threads, iters: int, a: float, b: float):
    """The reference's run_scaling_sweep + sweep_csv under its own synthetic
    timing model (tests/test_bench.cpp:142-150): (csv text, r_max, n08|None, C)."""
    L = _lib("reference")
    dims = np.ascontiguousarray(np.asarray(dims_list, dtype=np.int32).reshape(-1))
    thr = np.ascontiguousarray(np.asarray(threads, dtype=np.int32))
    buf = C.create_string_buffer(1 << 20)
    summ = np.zeros(3)
    _check(L, L.orc_sweep_model(int(bp[2]), p, dims.ctypes.data_as(C.POINTER(C.c_int)), len(dims_list),
                                thr.ctypes.data_as(C.POINTER(C.c_int)), len(threads), iters, a, b,
                                buf, len(buf), _dp(summ)))
    n08 = None if summ[1] < 0 else float(summ[1])
    return buf.value.decode(), float(summ[0]), n08, float(summ[2])


def record_json_reference(rec: dict) -> str:
    """The reference's bench_record_json (nlohmann::ordered_json dump)."""
    L = _lib("reference")
    buf = C.create_string_buffer(4096)
    _check(L, L.orc_record_json(rec["bp"].encode(), rec["p"], rec["q"], rec["E"], rec["n"], rec["P"],
                                rec["iterations"], rec["seconds"], rec["dofs_rate"], rec["n_per_rank"],
                                buf, len(buf)))
    return buf.value.decode()
