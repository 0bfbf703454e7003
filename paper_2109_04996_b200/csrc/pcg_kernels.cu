// Device-resident Jacobi-PCG: vector phases and fixed-order reductions.
//
// Restates the reference recurrence (proj/src/pcg.cpp:24-115) with every
// scalar kept on the device, three launches per iteration:
//   K1      Ap += A p over free rows (op_pencil.cuh / op_kernel.cuh); its last
//           CTA sums the p.(A p) partials + the constrained part and derives
//           alpha with the reference's checks (pcg.cpp:74-82)
//   update  x += alpha p, r -= alpha Ap; last CTA: ||r||, history,
//           convergence / limit (pcg.cpp:90-99), beta = rho' / rho
//   dir     p = r/d + beta p; Ap = (constrained ? p : 0), the next RED
//           target; last CTA: sum of p^2 on constrained rows
// Each reduction is per-CTA partials over a fixed grid summed in a fixed
// order by the CTA that finishes last ("last CTA" pattern, pcg_device.cuh):
// no extra launches, bitwise reproducible run to run (the reference's
// dot_deterministic, parallel.cpp:69-106, plays that role).  A kernel reads
// the stop flag only at its start; it is written only by a last CTA.

#include "pcg_device.cuh"
#include "pcg_kernels.h"

namespace hxf {

namespace {
constexpr int VT = 256;

__device__ __forceinline__ bool is_cons(const uint32_t* mask, int64_t node) {
  return mask && ((mask[node >> 5] >> (node & 31)) & 1u);
}
}  // namespace

__global__ void __launch_bounds__(VT)
    pcg_init_kernel(PcgState* st, int64_t n_L, int m, const double* __restrict__ b,
                    const double* __restrict__ d, double* __restrict__ dinv,
                    double* __restrict__ x, double* __restrict__ r,
                    double* __restrict__ p, double* __restrict__ Ap, const uint32_t* cons_mask,
                    double* part, double* hist) {
  __shared__ double scratch[VT / 32];
  double rr = 0.0, rz = 0.0, cc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int c = 0; c < m; ++c) {
    for (int64_t node = (int64_t)blockIdx.x * VT + threadIdx.x; node < n_L; node += stride) {
      const int64_t i = c * n_L + node;
      const double bi = b[i];
      double zi = bi;
      if (d) {
        const double di = 1.0 / d[i];  // Jacobi z = r / d as z = r * (1/d), once per solve
        dinv[i] = di;
        zi = bi * di;
      }
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
  const int g = gridDim.x;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[g + blockIdx.x] = s1;
    part[2 * g + blockIdx.x] = s2;
  }
  if (!pcg_last_cta(&st->counter[3])) return;
  const double tr = pcg_sum_partials<VT>(part, g, scratch);
  const double tz = pcg_sum_partials<VT>(part + g, g, scratch);
  const double tc = pcg_sum_partials<VT>(part + 2 * g, g, scratch);
  if (threadIdx.x == 0) {
    st->counter[3] = 0;
    const double norm_b = sqrt(tr);  // pcg.cpp:53-64
    st->it = 0;
    st->converged = 0;
    st->error = 0;
    st->stop = 0;
    st->cons_pp = tc;
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
    st->rho = tz;
  }
}

// Iteration `it` (1-based): x += alpha p, r -= alpha Ap; r.r, r.z partials;
// the last CTA decides convergence and beta.  VEC: 16-byte aligned vectors,
// two entries per 128-bit access, two pairs per loop trip.
template <bool VEC>
__global__ void __launch_bounds__(VT, 4)
    pcg_update_kernel(PcgState* st, int it, int64_t n, const double* __restrict__ d,
                      double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                      const double* __restrict__ Ap, double* part, double* hist) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double alpha = st->alpha;
  double rr = 0.0, rz = 0.0;
  const int64_t tid = (int64_t)blockIdx.x * VT + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * VT;
  auto one = [&](int64_t i) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    rr += ri * ri;
    rz += ri * (d ? ri * d[i] : ri);  // d holds 1/diag here
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
      rz += rv.x * (rv.x * dv.x) + rv.y * (rv.y * dv.y);  // dv = 1/diag (or 1)
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
  const int g = gridDim.x;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[g + blockIdx.x] = s1;
  }
  if (!pcg_last_cta(&st->counter[1])) return;
  const double trr = pcg_sum_partials<VT>(part, g, scratch);
  const double trz = pcg_sum_partials<VT>(part + g, g, scratch);
  if (threadIdx.x == 0) {
    st->counter[1] = 0;
    // pcg.cpp:90-107
    const double res = sqrt(trr);
    if (!isfinite(res)) {
      st->error = PCG_ERR_RESID;
      st->stop = 1;
      return;
    }
    st->it = it;
    st->res = res;
    hist[it] = res;
    const bool conv = res <= st->target;
    if (conv) st->converged = 1;
    if ((conv && !st->fixed) || it == st->limit || res == 0.0) {
      st->stop = 1;
      return;
    }
    st->beta = trz / st->rho;
    st->rho = trz;
  }
}

// p = z + beta p, Ap preset; last CTA sums p^2 over constrained rows.
// VEC: 16-byte aligned vectors and an even component stride n_L.
template <bool VEC>
__global__ void __launch_bounds__(VT, 4)
    pcg_direction_kernel(PcgState* st, int64_t n_L, int m, const double* __restrict__ d,
                         const double* __restrict__ r, double* __restrict__ p,
                         double* __restrict__ Ap, const uint32_t* cons_mask, double* part) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double beta = st->beta;
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
      auto two = [&](int64_t k, double2 rv, double2 pv, double2 dv) {
        double2 q;
        q.x = rv.x * dv.x + beta * pv.x;  // dv = 1/diag (or 1)
        q.y = rv.y * dv.y + beta * pv.y;
        p2[k] = q;
        const int64_t node = 2 * k;
        const uint32_t w = cons_mask ? (cons_mask[node >> 5] >> (node & 31)) & 3u : 0u;
        a2[k] = make_double2((w & 1u) ? q.x : 0.0, (w & 2u) ? q.y : 0.0);
        if (w & 1u) cc += q.x * q.x;
        if (w & 2u) cc += q.y * q.y;
      };
      const double2 one2 = make_double2(1.0, 1.0);
      int64_t k = tid;
      for (; k + stride < h; k += 2 * stride) {
        const int64_t k1 = k + stride;
        const double2 ra = r2[k], pa = p2[k], da = d ? d2[k] : one2;
        const double2 rb = r2[k1], pb = p2[k1], db = d ? d2[k1] : one2;
        two(k, ra, pa, da);
        two(k1, rb, pb, db);
      }
      if (k < h) two(k, r2[k], p2[k], d ? d2[k] : one2);
    } else {
      for (int64_t node = tid; node < n_L; node += stride) {
        const int64_t i = o + node;
        const double zi = d ? r[i] * d[i] : r[i];  // d holds 1/diag here
        const double pi = zi + beta * p[i];
        const bool cons = is_cons(cons_mask, node);
        p[i] = pi;
        Ap[i] = cons ? pi : 0.0;  // next RED target; constrained rows preset to A p = p
        if (cons) cc += pi * pi;
      }
    }
  }
  const double s = block_sum<VT>(cc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (!pcg_last_cta(&st->counter[2])) return;
  const double tc = pcg_sum_partials<VT>(part, gridDim.x, scratch);
  if (threadIdx.x == 0) {
    st->counter[2] = 0;
    st->cons_pp = tc;
  }
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
int vec_grid() { return num_sms() * 4; }

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

cudaError_t pcg_launch_init(cudaStream_t s, PcgState* st, int64_t n_L, int m, const double* b,
                            const double* d, double* dinv, double* x, double* r, double* p,
                            double* Ap, const uint32_t* mask, double* part, double* hist) {
  pcg_init_kernel<<<vec_grid(), VT, 0, s>>>(st, n_L, m, b, d, dinv, x, r, p, Ap, mask, part, hist);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int it, int64_t n, const double* d,
                              double* x, double* r, const double* p, const double* Ap,
                              double* part, double* hist) {
  if (aligned16(d) && aligned16(x) && aligned16(r) && aligned16(p) && aligned16(Ap))
    pcg_update_kernel<true><<<vec_grid(), VT, 0, s>>>(st, it, n, d, x, r, p, Ap, part, hist);
  else
    pcg_update_kernel<false><<<vec_grid(), VT, 0, s>>>(st, it, n, d, x, r, p, Ap, part, hist);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int64_t n_L, int m,
                                 const double* d, const double* r, double* p, double* Ap,
                                 const uint32_t* mask, double* part) {
  if ((n_L % 2) == 0 && aligned16(d) && aligned16(r) && aligned16(p) && aligned16(Ap))
    pcg_direction_kernel<true><<<vec_grid(), VT, 0, s>>>(st, n_L, m, d, r, p, Ap, mask, part);
  else
    pcg_direction_kernel<false><<<vec_grid(), VT, 0, s>>>(st, n_L, m, d, r, p, Ap, mask, part);
  count_launch();
  return cudaGetLastError();
}

}  // namespace hxf
