// Device-resident Jacobi-PCG: vector phases and fixed-order reductions.
//
// Restates the reference recurrence (proj/src/pcg.cpp:24-115) with every
// scalar kept on the device, three launches per iteration:
//   K1      Ap += A p over free rows (op_pencil.cuh / op_kernel.cuh) and
//           per-CTA partials of p.(A p)
//   update  [prologue] pAp = sum(K1 partials) + sum_{constrained} p^2, the
//           reference's checks (pcg.cpp:74-82), alpha = rho / pAp;
//           x += alpha p, r -= alpha Ap; partials of r.r and r.(r/d)
//   dir     [prologue] ||r||, history, convergence / limit (pcg.cpp:90-99),
//           beta = rho' / rho; p = r/d + beta p; Ap = (constrained ? p : 0),
//           the next RED target; partials of p^2 on constrained rows
// The prologues are computed REDUNDANTLY by every block from the same
// partials in the same fixed order, so all blocks agree on alpha / beta /
// stop without a separate finalize launch; block 0 publishes them.  Scalars
// a block reads at its start and the previous kernel wrote (rho) are
// double-buffered by iteration parity; the iteration index is a kernel
// argument.  Every reduction is per-CTA partials over a fixed grid summed in
// a fixed order: bitwise reproducible run to run (the reference's
// dot_deterministic, parallel.cpp:69-106, plays that role).
#include "hxf_device.cuh"
#include "pcg_kernels.h"

namespace hxf {

namespace {
constexpr int VT = 256;

__device__ __forceinline__ bool is_cons(const uint32_t* mask, int64_t node) {
  return mask && ((mask[node >> 5] >> (node & 31)) & 1u);
}

// Fixed-order sum of n partials by one block; result broadcast to all threads.
__device__ double block_reduce_all(const double* part, int n, double* scratch) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += VT) s += part[i];
  s = block_sum<VT>(s, scratch);
  if (threadIdx.x == 0) scratch[0] = s;
  __syncthreads();
  const double r = scratch[0];
  __syncthreads();
  return r;
}
}  // namespace

__global__ void __launch_bounds__(VT)
    pcg_init_kernel(int64_t n_L, int m, const double* __restrict__ b, const double* __restrict__ d,
                    double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                    double* __restrict__ Ap, const uint32_t* cons_mask, double* part) {
  __shared__ double scratch[VT / 32];
  double rr = 0.0, rz = 0.0, cc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int c = 0; c < m; ++c) {
    for (int64_t node = (int64_t)blockIdx.x * VT + threadIdx.x; node < n_L; node += stride) {
      const int64_t i = c * n_L + node;
      const double bi = b[i];
      const double zi = d ? bi / d[i] : bi;
      const bool cons = is_cons(cons_mask, node);
      x[i] = 0.0;
      r[i] = bi;
      p[i] = zi;
      Ap[i] = cons ? zi : 0.0;  // operator kernels skip constrained rows (A p = p there)
      rr += bi * bi;
      rz += bi * zi;
      if (cons) cc += zi * zi;
    }
  }
  const double s0 = block_sum<VT>(rr, scratch);
  const double s1 = block_sum<VT>(rz, scratch);
  const double s2 = block_sum<VT>(cc, scratch);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[gridDim.x + blockIdx.x] = s1;
    part[2 * gridDim.x + blockIdx.x] = s2;
  }
}

__global__ void __launch_bounds__(VT)
    pcg_init_finalize(PcgState* st, const double* part, int g, double* hist, double* cons_part) {
  __shared__ double scratch[VT / 32];
  const double rr = block_reduce_all(part, g, scratch);
  const double rz = block_reduce_all(part + g, g, scratch);
  const double cc = block_reduce_all(part + 2 * g, g, scratch);
  if (threadIdx.x == 0) {
    cons_part[0] = cc;  // read by the first update kernel as a 1-entry partial list
    const double norm_b = sqrt(rr);
    st->it = 0;
    st->converged = 0;
    st->error = 0;
    st->stop = 0;
    if (!isfinite(norm_b)) {
      st->error = PCG_ERR_RHS;
      st->stop = 1;
      return;
    }
    hist[0] = norm_b;
    st->norm_b = norm_b;
    st->res = norm_b;
    st->target = st->tol * norm_b;
    if (norm_b == 0.0) {
      st->converged = 1;
      st->stop = 1;
      return;
    }
    st->rho[1] = rz;  // rho before iteration 1
  }
}

// Iteration `it` (1-based): alpha prologue + x/r update + r.r, r.z partials.
// VEC: all vectors 16-byte aligned -> two entries per 128-bit access, two
// pairs per loop trip (more bytes in flight per thread).
template <bool VEC>
__global__ void __launch_bounds__(VT)
    pcg_update_kernel(PcgState* st, int it, const double* kpart, int gk, const double* cpart,
                      int gc, int64_t n, const double* __restrict__ d, double* __restrict__ x,
                      double* __restrict__ r, const double* __restrict__ p,
                      const double* __restrict__ Ap, double* part) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double pap = block_reduce_all(kpart, gk, scratch) + block_reduce_all(cpart, gc, scratch);
  const double rho = st->rho[it & 1];
  // pcg.cpp:74-82
  if (!isfinite(pap) || pap <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->pap = pap;
      if (!isfinite(pap)) st->error = PCG_ERR_APPLY_NAN;
      else if (rho == 0.0) st->converged = 1;
      else st->error = PCG_ERR_INDEFINITE;
      st->stop = 1;
    }
    return;
  }
  const double alpha = rho / pap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->pap = pap;
    st->alpha = alpha;
  }
  double rr = 0.0, rz = 0.0;
  const int64_t tid = (int64_t)blockIdx.x * VT + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * VT;
  auto one = [&](int64_t i) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    rr += ri * ri;
    rz += ri * (d ? ri / d[i] : ri);
  };
  if constexpr (VEC) {
    const int64_t n2 = n / 2;
    auto two = [&](int64_t k, double2 xv, double2 pv, double2 rv, double2 av, double2 dv) {
      xv.x += alpha * pv.x;
      xv.y += alpha * pv.y;
      rv.x -= alpha * av.x;
      rv.y -= alpha * av.y;
      reinterpret_cast<double2*>(x)[k] = xv;
      reinterpret_cast<double2*>(r)[k] = rv;
      rr += rv.x * rv.x + rv.y * rv.y;
      rz += rv.x * (d ? rv.x / dv.x : rv.x) + rv.y * (d ? rv.y / dv.y : rv.y);
    };
    const double2* x2 = reinterpret_cast<const double2*>(x);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* r2 = reinterpret_cast<const double2*>(r);
    const double2* a2 = reinterpret_cast<const double2*>(Ap);
    const double2* d2 = reinterpret_cast<const double2*>(d);
    const double2 one2 = make_double2(1.0, 1.0);
    int64_t k = tid;
    for (; k + stride < n2; k += 2 * stride) {
      const int64_t k1 = k + stride;
      const double2 xa = x2[k], pa = p2[k], ra = r2[k], aa = a2[k], da = d ? d2[k] : one2;
      const double2 xb = x2[k1], pb = p2[k1], rb = r2[k1], ab = a2[k1], db = d ? d2[k1] : one2;
      two(k, xa, pa, ra, aa, da);
      two(k1, xb, pb, rb, ab, db);
    }
    if (k < n2) two(k, x2[k], p2[k], r2[k], a2[k], d ? d2[k] : one2);
    if ((n & 1) && tid == 0) one(n - 1);
  } else {
    for (int64_t i = tid; i < n; i += stride) one(i);
  }
  const double s0 = block_sum<VT>(rr, scratch);
  const double s1 = block_sum<VT>(rz, scratch);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[gridDim.x + blockIdx.x] = s1;
  }
}

// Iteration `it`: residual / convergence prologue + p = z + beta p, Ap preset.
// VEC: 16-byte aligned vectors and an even component stride n_L.
template <bool VEC>
__global__ void __launch_bounds__(VT)
    pcg_direction_kernel(PcgState* st, int it, const double* upart, int gu, double* hist,
                         int64_t n_L, int m, const double* __restrict__ d,
                         const double* __restrict__ r, double* __restrict__ p,
                         double* __restrict__ Ap, const uint32_t* cons_mask, double* cpart) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double rr = block_reduce_all(upart, gu, scratch);
  const double rz = block_reduce_all(upart + gu, gu, scratch);
  const double res = sqrt(rr);
  const double rho = st->rho[it & 1];
  // pcg.cpp:90-107
  const bool bad = !isfinite(res);
  const bool conv = res <= st->target;
  const bool stop = bad || (conv && !st->fixed) || it == st->limit || res == 0.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (bad) {
      st->error = PCG_ERR_RESID;
    } else {
      st->it = it;
      st->res = res;
      hist[it] = res;
      if (conv) st->converged = 1;
    }
    if (!stop) {
      st->beta = rz / rho;
      st->rho[(it + 1) & 1] = rz;
    }
    st->stop = stop ? 1 : 0;
  }
  if (stop) return;
  const double beta = rz / rho;
  double cc = 0.0;
  const int64_t tid = (int64_t)blockIdx.x * VT + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int c = 0; c < m; ++c) {
    const int64_t o = c * n_L;
    if constexpr (VEC) {
      const int64_t h = n_L / 2;  // n_L even
      const double2* r2 = reinterpret_cast<const double2*>(r + o);
      const double2* d2 = reinterpret_cast<const double2*>(d + o);
      double2* p2 = reinterpret_cast<double2*>(p + o);
      double2* a2 = reinterpret_cast<double2*>(Ap + o);
      for (int64_t k = tid; k < h; k += stride) {
        const double2 rv = r2[k], pv = p2[k];
        const double2 dv = d ? d2[k] : make_double2(1.0, 1.0);
        double2 q;
        q.x = (d ? rv.x / dv.x : rv.x) + beta * pv.x;
        q.y = (d ? rv.y / dv.y : rv.y) + beta * pv.y;
        p2[k] = q;
        const int64_t node = 2 * k;
        const uint32_t w = cons_mask ? (cons_mask[node >> 5] >> (node & 31)) & 3u : 0u;
        a2[k] = make_double2((w & 1u) ? q.x : 0.0, (w & 2u) ? q.y : 0.0);
        if (w & 1u) cc += q.x * q.x;
        if (w & 2u) cc += q.y * q.y;
      }
    } else {
      for (int64_t node = tid; node < n_L; node += stride) {
        const int64_t i = o + node;
        const double zi = d ? r[i] / d[i] : r[i];
        const double pi = zi + beta * p[i];
        const bool cons = is_cons(cons_mask, node);
        p[i] = pi;
        Ap[i] = cons ? pi : 0.0;  // next RED target; constrained rows preset to A p = p
        if (cons) cc += pi * pi;
      }
    }
  }
  const double s = block_sum<VT>(cc, scratch);
  if (threadIdx.x == 0) cpart[blockIdx.x] = s;
}

// y = x on constrained rows, 0 elsewhere: the RED target of an operator apply
// (operator.cpp:87-90,141-143).
__global__ void __launch_bounds__(VT)
    init_y_kernel(int64_t n_L, int m, const double* __restrict__ x, double* __restrict__ y,
                  const uint32_t* cons_mask) {
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int c = 0; c < m; ++c)
    for (int64_t node = (int64_t)blockIdx.x * VT + threadIdx.x; node < n_L; node += stride) {
      const int64_t i = c * n_L + node;
      y[i] = is_cons(cons_mask, node) ? x[i] : 0.0;
    }
}

// ------------------------------------------------------------------ host side
int vec_grid() { return num_sms() * 8; }

namespace {
bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}  // namespace

cudaError_t launch_init_y(cudaStream_t s, int64_t n_L, int m, const double* x, double* y,
                          const uint32_t* mask) {
  if (!mask) return cudaMemsetAsync(y, 0, sizeof(double) * n_L * m, s);
  init_y_kernel<<<vec_grid(), VT, 0, s>>>(n_L, m, x, y, mask);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_init(cudaStream_t s, int64_t n_L, int m, const double* b, const double* d,
                            double* x, double* r, double* p, double* Ap, const uint32_t* mask,
                            double* part, PcgState* st, double* hist, double* cons_part) {
  const int g = vec_grid();
  pcg_init_kernel<<<g, VT, 0, s>>>(n_L, m, b, d, x, r, p, Ap, mask, part);
  pcg_init_finalize<<<1, VT, 0, s>>>(st, part, g, hist, cons_part);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int it, const double* kpart, int gk,
                              const double* cpart, int gc, int64_t n, const double* d, double* x,
                              double* r, const double* p, const double* Ap, double* upart) {
  if (aligned16(d) && aligned16(x) && aligned16(r) && aligned16(p) && aligned16(Ap))
    pcg_update_kernel<true><<<vec_grid(), VT, 0, s>>>(st, it, kpart, gk, cpart, gc, n, d, x, r, p,
                                                     Ap, upart);
  else
    pcg_update_kernel<false><<<vec_grid(), VT, 0, s>>>(st, it, kpart, gk, cpart, gc, n, d, x, r,
                                                      p, Ap, upart);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int it, const double* upart,
                                 double* hist, int64_t n_L, int m, const double* d,
                                 const double* r, double* p, double* Ap, const uint32_t* mask,
                                 double* cpart) {
  if ((n_L % 2) == 0 && aligned16(d) && aligned16(r) && aligned16(p) && aligned16(Ap))
    pcg_direction_kernel<true><<<vec_grid(), VT, 0, s>>>(st, it, upart, vec_grid(), hist, n_L, m,
                                                        d, r, p, Ap, mask, cpart);
  else
    pcg_direction_kernel<false><<<vec_grid(), VT, 0, s>>>(st, it, upart, vec_grid(), hist, n_L, m,
                                                         d, r, p, Ap, mask, cpart);
  count_launch();
  return cudaGetLastError();
}

}  // namespace hxf
