// K2-K4: device-resident Jacobi-PCG vector phases and fixed-order reductions.
//
// Restates the reference recurrence (proj/src/pcg.cpp:24-115) with the
// scalars kept on the device (PcgState) so a whole solve runs without a host
// round trip per iteration:
//   init     x = 0, r = b, p = z = b/d, partials of b.b and b.z
//   K1       Ap = A p (op_kernel.cuh) + partials of p.Ap over free nodes
//   alpha    pAp = sum(partials) + sum_{constrained} p^2; checks; alpha
//   update   x += alpha p, r -= alpha Ap; partials of r.r and r.(r/d)
//   resid    ||r||, history, convergence / limit; beta = rho'/rho
//   dir      p = r/d + beta p; Ap = 0 (next RED target); partials of p^2 on
//            constrained nodes
// Every reduction is per-CTA partials (fixed grid) summed in a fixed order by
// one block: bitwise reproducible run to run for a fixed launch geometry
// (the reference's dot_deterministic, parallel.cpp:69-106, plays that role).
#include "hxf_device.cuh"
#include "pcg_kernels.h"

namespace hxf {

namespace {
constexpr int VT = 256;

__device__ __forceinline__ bool is_cons(const uint32_t* mask, int64_t node) {
  return mask && ((mask[node >> 5] >> (node & 31)) & 1u);
}

// Fixed-order sum of `n` partials with stride `stride`, one block of VT threads.
__device__ double reduce_partials(const double* part, int n, double* scratch) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += VT) s += part[i];
  return block_sum<VT>(s, scratch);  // valid on thread 0
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
    pcg_init_finalize(PcgState* st, const double* part, int g, double* hist) {
  __shared__ double scratch[VT / 32];
  const double rr = reduce_partials(part, g, scratch);
  const double rz = reduce_partials(part + g, g, scratch);
  const double cc = reduce_partials(part + 2 * g, g, scratch);
  if (threadIdx.x == 0) {
    const double norm_b = sqrt(rr);
    st->it = 0;
    st->converged = 0;
    st->error = 0;
    st->stop = 0;
    st->cons_pp = cc;
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
    st->rho = rz;
  }
}

__global__ void __launch_bounds__(VT)
    pcg_alpha_finalize(PcgState* st, const double* kpart, int gk) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double s = reduce_partials(kpart, gk, scratch);
  if (threadIdx.x == 0) {
    const double pap = s + st->cons_pp;
    st->pap = pap;
    if (!isfinite(pap)) {
      st->error = PCG_ERR_APPLY_NAN;
      st->stop = 1;
      return;
    }
    if (pap <= 0.0) {
      if (st->rho == 0.0) {
        st->converged = 1;
      } else {
        st->error = PCG_ERR_INDEFINITE;
      }
      st->stop = 1;
      return;
    }
    st->alpha = st->rho / pap;
  }
}

__global__ void __launch_bounds__(VT)
    pcg_update_kernel(const PcgState* st, int64_t n, const double* __restrict__ d,
                      double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                      const double* __restrict__ Ap, double* part) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double alpha = st->alpha;
  double rr = 0.0, rz = 0.0;
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int64_t i = (int64_t)blockIdx.x * VT + threadIdx.x; i < n; i += stride) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * Ap[i];
    r[i] = ri;
    rr += ri * ri;
    rz += ri * (d ? ri / d[i] : ri);
  }
  const double s0 = block_sum<VT>(rr, scratch);
  const double s1 = block_sum<VT>(rz, scratch);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[gridDim.x + blockIdx.x] = s1;
  }
}

__global__ void __launch_bounds__(VT)
    pcg_update_finalize(PcgState* st, const double* part, int g, double* hist) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double rr = reduce_partials(part, g, scratch);
  const double rz = reduce_partials(part + g, g, scratch);
  if (threadIdx.x == 0) {
    const double res = sqrt(rr);
    if (!isfinite(res)) {
      st->error = PCG_ERR_RESID;
      st->stop = 1;
      return;
    }
    const int it = st->it + 1;
    st->it = it;
    st->res = res;
    hist[it] = res;
    if (res <= st->target) {
      st->converged = 1;
      if (!st->fixed) st->stop = 1;
    }
    if (it == st->limit || res == 0.0) st->stop = 1;
    if (st->stop) return;
    st->beta = rz / st->rho;
    st->rho = rz;
  }
}

__global__ void __launch_bounds__(VT)
    pcg_direction_kernel(PcgState* st, int64_t n_L, int m, const double* __restrict__ d,
                         const double* __restrict__ r, double* __restrict__ p,
                         double* __restrict__ Ap, const uint32_t* cons_mask, double* part) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double beta = st->beta;
  double cc = 0.0;
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int c = 0; c < m; ++c) {
    for (int64_t node = (int64_t)blockIdx.x * VT + threadIdx.x; node < n_L; node += stride) {
      const int64_t i = c * n_L + node;
      const double zi = d ? r[i] / d[i] : r[i];
      const double pi = zi + beta * p[i];
      const bool cons = is_cons(cons_mask, node);
      p[i] = pi;
      Ap[i] = cons ? pi : 0.0;  // next RED target; constrained rows preset to A p = p
      if (cons) cc += pi * pi;
    }
  }
  if (cons_mask) {
    const double s = block_sum<VT>(cc, scratch);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(VT)
    pcg_cons_finalize(PcgState* st, const double* part, int g) {
  __shared__ double scratch[VT / 32];
  if (st->stop) return;
  const double s = reduce_partials(part, g, scratch);
  if (threadIdx.x == 0) st->cons_pp = s;
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

cudaError_t pcg_launch_init(cudaStream_t s, int64_t n_L, int m, const double* b, const double* d,
                            double* x, double* r, double* p, double* Ap, const uint32_t* mask,
                            double* part, PcgState* st, double* hist) {
  const int g = vec_grid();
  pcg_init_kernel<<<g, VT, 0, s>>>(n_L, m, b, d, x, r, p, Ap, mask, part);
  pcg_init_finalize<<<1, VT, 0, s>>>(st, part, g, hist);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t launch_init_y(cudaStream_t s, int64_t n_L, int m, const double* x, double* y,
                          const uint32_t* mask) {
  if (!mask) return cudaMemsetAsync(y, 0, sizeof(double) * n_L * m, s);
  init_y_kernel<<<vec_grid(), VT, 0, s>>>(n_L, m, x, y, mask);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_alpha(cudaStream_t s, PcgState* st, const double* kpart, int gk) {
  pcg_alpha_finalize<<<1, VT, 0, s>>>(st, kpart, gk);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int64_t n, const double* d, double* x,
                              double* r, const double* p, const double* Ap, double* part,
                              double* hist) {
  const int g = vec_grid();
  pcg_update_kernel<<<g, VT, 0, s>>>(st, n, d, x, r, p, Ap, part);
  pcg_update_finalize<<<1, VT, 0, s>>>(st, part, g, hist);
  count_launch(2);
  return cudaGetLastError();
}

cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int64_t n_L, int m,
                                 const double* d, const double* r, double* p, double* Ap,
                                 const uint32_t* mask, double* part) {
  const int g = vec_grid();
  pcg_direction_kernel<<<g, VT, 0, s>>>(st, n_L, m, d, r, p, Ap, mask, part);
  count_launch();
  if (mask) {
    pcg_cons_finalize<<<1, VT, 0, s>>>(st, part, g);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace hxf
