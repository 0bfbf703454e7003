// Device-resident Jacobi-PCG: vector phases and fixed-order reductions.
//
// Restates the reference recurrence (proj/src/pcg.cpp:24-115) with every
// scalar kept on the device, three launches per iteration:
//   K1      Ap += A p over free rows (op_dmma / op_pencil / op_kernel); its
//           last CTA writes this rank's pAp into red[0]
//   update  every CTA derives alpha = rho / pAp from red[0] with the
//           reference's checks (pcg.cpp:74-82); r -= alpha Ap;
//           last CTA: red[1] = r.r, red[2] = r.(r/d) over owned rows
//   dir     x += alpha p (pcg.cpp:84-88: moved here, where p is read anyway —
//           one vector pass less per iteration; x is still updated before
//           the loop can stop); every CTA derives ||r||, convergence / limit
//           (pcg.cpp:90-99) and beta = rho' / rho from red[1..2]; unless
//           stopping, p = r/d + beta p and Ap = (constrained & owned ? p : 0),
//           the next RED target; the last CTA records the iteration (or the
//           stop) and red[3] = sum of p^2 over owned constrained rows
// On a partitioned problem red[] is all-reduced across ranks between the
// kernels (dist.cu); on one GPU the same kernels run back to back.  Each
// reduction is per-CTA partials over a fixed grid summed in a fixed order by
// the CTA that finishes last (pcg_device.cuh): bitwise reproducible run to
// run (the reference's dot_deterministic, parallel.cpp:69-106, plays that
// role).  Scalars are read at kernel start and written only by the last CTA
// (or, on an early stop, by CTA 0 — nothing reads them later in that kernel).
#include <cstdlib>

#include "pcg_device.cuh"
#include "pcg_kernels.h"

namespace hxf {

namespace {
constexpr int VT = 256;

__device__ __forceinline__ uint32_t bit_of(const uint32_t* mask, int64_t node) {
  return (mask[node >> 5] >> (node & 31)) & 1u;
}
__device__ __forceinline__ bool is_cons(const uint32_t* mask, int64_t node) {
  return mask && bit_of(mask, node);
}
// owned rows weigh 1 in dots (no owner mask: everything is owned)
__device__ __forceinline__ double owned_w(const uint32_t* own, int64_t node) {
  return (!own || bit_of(own, node)) ? 1.0 : 0.0;
}
}  // namespace

__global__ void __launch_bounds__(VT)
    pcg_init_kernel(PcgState* st, int64_t n_L, int m, const double* __restrict__ b,
                    const double* __restrict__ d, double* __restrict__ dinv,
                    double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                    double* __restrict__ Ap, const uint32_t* cons_mask, const uint32_t* own,
                    double* part) {
  __shared__ double scratch[VT / 32];
  double bb = 0.0, bz = 0.0, cc = 0.0;
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
      const double w = owned_w(own, node);
      const bool cons = is_cons(cons_mask, node);
      x[i] = 0.0;
      r[i] = bi;
      p[i] = zi;
      // operator kernels skip constrained rows (A p = p there); one owner
      // presets it so an interface sum-exchange leaves exactly p
      Ap[i] = (cons && w != 0.0) ? zi : 0.0;
      bb += w * bi * bi;
      bz += w * bi * zi;
      if (cons) cc += w * zi * zi;
    }
  }
  const double s0 = block_sum<VT>(bb, scratch);
  const double s1 = block_sum<VT>(bz, scratch);
  const double s2 = block_sum<VT>(cc, scratch);
  const int g = gridDim.x;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = s0;
    part[g + blockIdx.x] = s1;
    part[2 * g + blockIdx.x] = s2;
  }
  if (!pcg_last_cta(&st->counter[3])) return;
  const double tb = pcg_sum_partials<VT>(part, g, scratch);
  const double tz = pcg_sum_partials<VT>(part + g, g, scratch);
  const double tc = pcg_sum_partials<VT>(part + 2 * g, g, scratch);
  if (threadIdx.x == 0) {
    st->counter[3] = 0;
    st->red[3] = tc;  // stays local: K1 adds it before its own all-reduce
    st->red[4] = tb;
    st->red[5] = tz;
  }
}

// After (optionally) all-reducing red[4..5]: ||b||, rho, checks (pcg.cpp:53-64).
__global__ void pcg_init_finalize(PcgState* st, double* hist) {
  if (threadIdx.x != 0) return;
  const double norm_b = sqrt(st->red[4]);
  st->it = 0;
  st->converged = 0;
  st->error = 0;
  st->stop = 0;
  st->stop_update = 0;
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
  st->rho = st->red[5];
}

// Iteration `it` (1-based).  VEC: 16-byte aligned vectors, even n_L, two
// entries per 128-bit access, two pairs per loop trip.  OWN: owner-weighted
// dots (partitioned); a separate instantiation keeps the single-domain loop
// within 64 registers.
template <bool VEC, bool OWN>
__global__ void __launch_bounds__(VT, OWN ? 3 : 4)
    pcg_update_kernel(PcgState* st, int it, int64_t n_L, int m, const double* __restrict__ d,
                      double* __restrict__ r, const double* __restrict__ Ap, const uint32_t* own,
                      double* part, int rev) {
  __shared__ double scratch[VT / 32];
  pdl_wait();
  if (st->stop) return;
  const double pap = st->red[0];
  const double rho = st->rho;
  // pcg.cpp:74-82
  if (!isfinite(pap) || pap <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->pap = pap;
      if (!isfinite(pap)) st->error = PCG_ERR_APPLY_NAN;
      else if (rho == 0.0) st->converged = 1;
      else st->error = PCG_ERR_INDEFINITE;
      st->stop_update = it;
      st->stop = 1;
    }
    return;
  }
  const double alpha = rho / pap;
  double rr = 0.0, rz = 0.0;
  const int64_t tid = (int64_t)blockIdx.x * VT + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * VT;
  // without an owner mask nothing depends on the node: one flat pass
  const int mc = OWN ? m : 1;
  if constexpr (!OWN) n_L *= m;
  for (int c = 0; c < mc; ++c) {
    const int64_t o = c * n_L;
    if constexpr (VEC) {
      const int64_t h = n_L / 2;
      double2* r2 = reinterpret_cast<double2*>(r + o);
      const double2* a2 = reinterpret_cast<const double2*>(Ap + o);
      const double2* d2 = reinterpret_cast<const double2*>(d + o);
      const double2 one2 = make_double2(1.0, 1.0);
      auto two = [&](int64_t k, double2 rv, double2 av, double2 dv) {
        // (k is already the swept pair index)
        rv.x -= alpha * av.x;
        rv.y -= alpha * av.y;
        r2[k] = rv;
        const int64_t node = 2 * k;
        if constexpr (OWN) {
          const uint32_t wb = (own[node >> 5] >> (node & 31)) & 3u;
          const double w0 = (wb & 1u) ? 1.0 : 0.0, w1 = (wb & 2u) ? 1.0 : 0.0;
          rr += w0 * rv.x * rv.x + w1 * rv.y * rv.y;
          rz += w0 * rv.x * (rv.x * dv.x) + w1 * rv.y * (rv.y * dv.y);  // dv = 1/diag (or 1)
        } else {
          rr += rv.x * rv.x + rv.y * rv.y;
          rz += rv.x * (rv.x * dv.x) + rv.y * (rv.y * dv.y);
        }
      };
      int64_t j = tid;
      for (; j + stride < h; j += 2 * stride) {
        const int64_t k = rev ? h - 1 - j : j, k1 = rev ? k - stride : k + stride;
        const double2 ra = r2[k], aa = a2[k], da = d ? d2[k] : one2;
        const double2 rb = r2[k1], ab = a2[k1], db = d ? d2[k1] : one2;
        two(k, ra, aa, da);
        two(k1, rb, ab, db);
      }
      if (j < h) {
        const int64_t k = rev ? h - 1 - j : j;
        two(k, r2[k], a2[k], d ? d2[k] : one2);
      }
    } else {
      for (int64_t jn = tid; jn < n_L; jn += stride) {
        const int64_t node = rev ? n_L - 1 - jn : jn;
        const int64_t i = o + node;
        const double ri = r[i] - alpha * Ap[i];
        r[i] = ri;
        const double w = OWN ? owned_w(own, node) : 1.0;
        rr += w * ri * ri;
        rz += w * ri * (d ? ri * d[i] : ri);  // d holds 1/diag here
      }
    }
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
    st->pap = pap;
    st->alpha = alpha;
    st->red[1] = trr;
    st->red[2] = trz;
  }
}

// Iteration `it`: residual / convergence from red[1..2] (pcg.cpp:90-107);
// p = z + beta p, Ap preset.  VEC: as for the update kernel.
template <bool VEC>
__global__ void __launch_bounds__(VT, 4)
    pcg_direction_kernel(PcgState* st, int it, double* hist, int64_t n_L, int m,
                         const double* __restrict__ d, const double* __restrict__ r,
                         double* __restrict__ x, const double* p, const double* pprev, double* pout,
                         double* __restrict__ Ap, const uint32_t* cons_mask, const uint32_t* own,
                         double* part, int rev, int xmode) {
  __shared__ double scratch[VT / 32];
  pdl_wait();
  if (st->stop) {
    // stopped by the update kernel (pAp check, pcg.cpp:74-82): x gets only the
    // update still pending from the previous iteration (batched mode)
    // (only when this iteration's update stopped: kernels of iterations
    // enqueued past an earlier stop must leave x alone)
    if (xmode == 2 && !st->error && st->stop_update == it) {
      const double ap = st->alpha_prev;
      const int64_t n = n_L * m, stride = (int64_t)gridDim.x * VT;
      for (int64_t i = (int64_t)blockIdx.x * VT + threadIdx.x; i < n; i += stride)
        x[i] = fma(ap, pprev[i], x[i]);
    }
    return;
  }
  const double alpha = st->alpha;
  // xmode 0: x += alpha p; 1: deferred to the next iteration (unless
  // stopping); 2: x += alpha_prev p_prev + alpha p (same rounding sequence as
  // two single updates: x <- fma(alpha, p, fma(alpha_prev, p_prev, x)))
  const double alpha_prev = xmode == 2 ? st->alpha_prev : 0.0;
  const double rr = st->red[1], rz = st->red[2];
  const double res = sqrt(rr);
  const double rho = st->rho;
  const bool bad = !isfinite(res);
  const bool conv = res <= st->target;
  // stopping: only x += alpha p below; the last CTA publishes the stop (no
  // CTA may see st->stop set before it has done its part of x)
  const bool stop = bad || (conv && !st->fixed) || it == st->limit || res == 0.0;
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
      const double2* p2 = reinterpret_cast<const double2*>(p + o);
      const double2* pp2 = reinterpret_cast<const double2*>((xmode == 2 ? pprev : p) + o);
      double2* po2 = reinterpret_cast<double2*>(pout + o);
      double2* a2 = reinterpret_cast<double2*>(Ap + o);
      double2* x2 = reinterpret_cast<double2*>(x + o);
      const bool xupd = xmode != 1 || stop;
      auto two = [&](int64_t k, double2 rv, double2 pv, double2 dv) {
        if (xupd) {
          double2 xv = x2[k];
          if (xmode == 2) {
            const double2 qv = pp2[k];
            xv.x = fma(alpha_prev, qv.x, xv.x);
            xv.y = fma(alpha_prev, qv.y, xv.y);
          }
          xv.x = fma(alpha, pv.x, xv.x);
          xv.y = fma(alpha, pv.y, xv.y);
          x2[k] = xv;
        }
        if (stop) return;
        double2 q;
        q.x = rv.x * dv.x + beta * pv.x;  // dv = 1/diag (or 1)
        q.y = rv.y * dv.y + beta * pv.y;
        po2[k] = q;
        const int64_t node = 2 * k;
        uint32_t w = cons_mask ? (cons_mask[node >> 5] >> (node & 31)) & 3u : 0u;
        if (own) w &= (own[node >> 5] >> (node & 31)) & 3u;
        a2[k] = make_double2((w & 1u) ? q.x : 0.0, (w & 2u) ? q.y : 0.0);
        if (w & 1u) cc += q.x * q.x;
        if (w & 2u) cc += q.y * q.y;
      };
      const double2 one2 = make_double2(1.0, 1.0);
      int64_t j = tid;
      for (; j + stride < h; j += 2 * stride) {
        const int64_t k = rev ? h - 1 - j : j, k1 = rev ? k - stride : k + stride;
        const double2 pa = p2[k], pb = p2[k1];
        const double2 ra = stop ? one2 : r2[k], da = (d && !stop) ? d2[k] : one2;
        const double2 rb = stop ? one2 : r2[k1], db = (d && !stop) ? d2[k1] : one2;
        two(k, ra, pa, da);
        two(k1, rb, pb, db);
      }
      if (j < h) {
        const int64_t k = rev ? h - 1 - j : j;
        two(k, stop ? one2 : r2[k], p2[k], (d && !stop) ? d2[k] : one2);
      }
    } else {
      for (int64_t jn = tid; jn < n_L; jn += stride) {
        const int64_t node = rev ? n_L - 1 - jn : jn;
        const int64_t i = o + node;
        const double po = p[i];
        if (xmode != 1 || stop) {
          double xv = x[i];
          if (xmode == 2) xv = fma(alpha_prev, pprev[i], xv);
          x[i] = fma(alpha, po, xv);
        }
        if (stop) continue;
        const double zi = d ? r[i] * d[i] : r[i];  // d holds 1/diag here
        const double pi = zi + beta * po;
        const bool cw = is_cons(cons_mask, node) && owned_w(own, node) != 0.0;
        pout[i] = pi;
        Ap[i] = cw ? pi : 0.0;  // next RED target; constrained rows preset to A p = p
        if (cw) cc += pi * pi;
      }
    }
  }
  const double s = block_sum<VT>(cc, scratch);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
  if (!pcg_last_cta(&st->counter[2])) return;
  const double tc = pcg_sum_partials<VT>(part, gridDim.x, scratch);
  if (threadIdx.x == 0) {
    st->counter[2] = 0;
    if (stop) {
      if (bad) {
        st->error = PCG_ERR_RESID;
      } else {
        st->it = it;
        st->res = res;
        hist[it] = res;
        if (conv) st->converged = 1;
      }
      st->stop = 1;
      return;
    }
    st->red[3] = tc;
    st->it = it;
    st->res = res;
    hist[it] = res;
    if (conv) st->converged = 1;
    st->beta = beta;
    st->rho = rz;
    st->alpha_prev = alpha;
  }
}

// ---------------------------------------------------------------- fused step
// Update and direction of iteration `it` in one persistent cooperative kernel
// (single domain, one CTA per SM): phase 1 is the update kernel's
// r -= alpha Ap with the r.r / r.z partials over grid-stride steps, z = r/d of
// the CTA's first zcap pairs kept in shared memory; a grid barrier; every CTA
// sums the partials in the same fixed order (same bits everywhere); phase 2
// is the direction kernel over the same pairs in the opposite step order (the
// windows phase 1 touched last, still in L2, first; then the cached z).
// Saves the r and 1/d re-reads of the cached pairs (2/3 of the vectors at C3)
// and one kernel boundary per iteration.
constexpr int ST_NT = 1024;
// measurement-only phase timestamps of the fused step kernel (tools/step_phases.py)
__device__ unsigned long long g_step_ts[4][1024];
__device__ int g_step_ts_on;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
constexpr int ST_SMEM = 192 * 1024;

__device__ __forceinline__ void grid_barrier(unsigned int* count, unsigned int* gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = gen;
    const unsigned int g0 = *vgen;
    __threadfence();
    if (atomicAdd(count, 1u) == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(gen, 1u);
    } else {
      while (*vgen == g0) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// ST_CS: the x and r stores evict-first (written back to HBM while this kernel
// runs instead of being flushed under the next operator kernel)
// ST_U / ST_U2: grid-stride steps per loop trip of phase 1 / 2 (loads of all
// of them first: phase 2 of an odd iteration has one global load per step)
template <int ST_U, int ST_U2, int ST_CS>
__global__ void __launch_bounds__(ST_NT, 1)
    pcg_step_kernel(PcgState* st, int it, double* hist, int64_t n_L, int m,
                    const double* __restrict__ d, double* __restrict__ r, double* __restrict__ x,
                    const double* p, const double* pprev, double* pout, double* __restrict__ Ap,
                    const uint32_t* cons_mask, double* part, int rev, int xmode, int ap_zero) {
  extern __shared__ double2 zc[];
  __shared__ double scratch[ST_NT / 32];
  constexpr int zcap = ST_SMEM / 16;
  if (st->stop) return;  // stopped in an earlier iteration
  const bool ts = g_step_ts_on == it && threadIdx.x == 0;  // (iteration to stamp)
  if (ts) g_step_ts[0][blockIdx.x] = gtimer();
  const double pap = st->red[0];
  const double rho = st->rho;
  const int G = gridDim.x;
  const int64_t h = n_L * m / 2;  // pairs (n_L even)
  // grid-stride steps j: the CTA's pair of step j (phase-1 order; -1 past the
  // end) — every step is one contiguous window of the vectors, so each phase
  // sweeps them (serpentine L2 reuse with the operator kernels as before)
  // (32-bit pair indices: the launcher requires h < 2^31)
  const int hh = (int)h;
  const int span = G * ST_NT;
  const int nj = (hh + span - 1) / span;
  auto pair_at = [&](int j) -> int {
    const int k = (j * G + (int)blockIdx.x) * ST_NT + (int)threadIdx.x;
    return k < hh ? (rev ? hh - 1 - k : k) : -1;
  };
  double2* x2 = reinterpret_cast<double2*>(x);
  const double alpha_prev = xmode == 2 ? st->alpha_prev : 0.0;
  // pcg.cpp:74-82 (as pcg_update_kernel) and, on a stop there, the pending
  // batched x update (as pcg_direction_kernel's stopped branch)
  if (!isfinite(pap) || pap <= 0.0) {
    const bool err = !isfinite(pap) || rho != 0.0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      st->pap = pap;
      if (!isfinite(pap)) st->error = PCG_ERR_APPLY_NAN;
      else if (rho == 0.0) st->converged = 1;
      else st->error = PCG_ERR_INDEFINITE;
      st->stop_update = it;
      st->stop = 1;
    }
    if (xmode == 2 && !err) {
      const double2* q2 = reinterpret_cast<const double2*>(pprev);
      for (int j = 0; j < nj; ++j) {
        const int k = pair_at(j);
        if (k < 0) continue;
        double2 xv = x2[k];
        const double2 pv = q2[k];
        xv.x = fma(alpha_prev, pv.x, xv.x);
        xv.y = fma(alpha_prev, pv.y, xv.y);
        x2[k] = xv;
      }
    }
    return;
  }
  const double alpha = rho / pap;
  const double2 one2 = make_double2(1.0, 1.0);
  double2* r2 = reinterpret_cast<double2*>(r);
  const double2* d2 = reinterpret_cast<const double2*>(d);
  double2* a2 = reinterpret_cast<double2*>(Ap);

  // ---- phase 1: r -= alpha Ap; r.r, r.z (pcg.cpp:84-88) ----
  // (ST_U steps per trip, loads first: enough bytes in flight at one CTA per SM)
  double rr = 0.0, rz = 0.0;
  for (int j0 = 0; j0 < nj; j0 += ST_U) {
    int k[ST_U];
    double2 rv[ST_U], av[ST_U], dv[ST_U];
#pragma unroll
    for (int u = 0; u < ST_U; ++u) {
      k[u] = j0 + u < nj ? pair_at(j0 + u) : -1;
      if (k[u] >= 0) {
        rv[u] = r2[k[u]];
        av[u] = a2[k[u]];
        dv[u] = d ? d2[k[u]] : one2;
      }
    }
#pragma unroll
    for (int u = 0; u < ST_U; ++u) {
      if (k[u] < 0) continue;
      double2 v = rv[u];
      v.x -= alpha * av[u].x;
      v.y -= alpha * av[u].y;
      if (ST_CS) __stcs(r2 + k[u], v); else r2[k[u]] = v;
      if (ap_zero) a2[k[u]] = make_double2(0.0, 0.0);  // the next operator kernel's RED target
      const double2 z = make_double2(v.x * dv[u].x, v.y * dv[u].y);
      rr += v.x * v.x + v.y * v.y;
      rz += v.x * z.x + v.y * z.y;
      const int q = (j0 + u) * ST_NT + (int)threadIdx.x;
      if (q < zcap) zc[q] = z;
    }
  }
  {
    const double s0 = block_sum<ST_NT>(rr, scratch);
    const double s1 = block_sum<ST_NT>(rz, scratch);
    if (threadIdx.x == 0) {
      part[blockIdx.x] = s0;
      part[G + blockIdx.x] = s1;
    }
  }
  if (ts) g_step_ts[1][blockIdx.x] = gtimer();
  grid_barrier(&st->gbar[0], &st->gbar[1]);
  if (ts) g_step_ts[2][blockIdx.x] = gtimer();
  __shared__ double tot[2];
  {
    const double trr = pcg_sum_partials<ST_NT>(part, G, scratch);
    const double trz = pcg_sum_partials<ST_NT>(part + G, G, scratch);
    if (threadIdx.x == 0) {
      tot[0] = trr;
      tot[1] = trz;
    }
    __syncthreads();
  }
  const double trr = tot[0], trz = tot[1];

  // ---- phase 2: convergence (pcg.cpp:90-99), x += alpha p, p = z + beta p,
  //      Ap preset (as pcg_direction_kernel) ----
  const double res = sqrt(trr);
  const bool bad = !isfinite(res);
  const bool conv = res <= st->target;
  const bool stop = bad || (conv && !st->fixed) || it == st->limit || res == 0.0;
  const double beta = trz / rho;
  const bool xupd = xmode != 1 || stop;
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* pp2 = reinterpret_cast<const double2*>(xmode == 2 ? pprev : p);
  double2* po2 = reinterpret_cast<double2*>(pout);
  double cc = 0.0;
  // one direction step: x update (xmode), p = z + beta p, Ap preset, cc
  auto dir_step = [&](int j, int kk, double2 pv, double2 xv, double2 qv) {
    if (xupd) {
      double2 xn = xv;
      if (xmode == 2) {
        xn.x = fma(alpha_prev, qv.x, xn.x);
        xn.y = fma(alpha_prev, qv.y, xn.y);
      }
      xn.x = fma(alpha, pv.x, xn.x);
      xn.y = fma(alpha, pv.y, xn.y);
      if (ST_CS) __stcs(x2 + kk, xn); else x2[kk] = xn;
    }
    if (stop) return;
    const int q = j * ST_NT + (int)threadIdx.x;
    double2 z;
    if (q < zcap) {
      z = zc[q];
    } else {
      const double2 rv = r2[kk], dv = d ? d2[kk] : one2;
      z = make_double2(rv.x * dv.x, rv.y * dv.y);
    }
    double2 pn;
    pn.x = z.x + beta * pv.x;
    pn.y = z.y + beta * pv.y;
    if (ST_CS >= 2) __stcs(po2 + kk, pn); else po2[kk] = pn;
    int64_t node = 2 * (int64_t)kk;
    for (int c = 1; c < m && node >= n_L; ++c) node -= n_L;  // component offset (no division)
    const uint32_t w = cons_mask ? (cons_mask[node >> 5] >> (node & 31)) & 3u : 0u;
    if (!ap_zero) {
      const double2 av = make_double2((w & 1u) ? pn.x : 0.0, (w & 2u) ? pn.y : 0.0);
      if (ST_CS >= 3) __stcs(a2 + kk, av); else a2[kk] = av;
    }
    if (w & 1u) cc += pn.x * pn.x;
    if (w & 2u) cc += pn.y * pn.y;
  };
  if constexpr (ST_U2 == 0) {
    // the next step's p (and x, p_prev) loaded before this step is processed
    const double2 zero2 = make_double2(0.0, 0.0);
    int kc = pair_at(nj - 1);
    double2 pc = zero2, xc = zero2, qc = zero2;
    if (kc >= 0) {
      pc = p2[kc];
      if (xupd) xc = x2[kc];
      if (xupd && xmode == 2) qc = pp2[kc];
    }
    for (int j = nj - 1; j >= 0; --j) {
      const int kn = j > 0 ? pair_at(j - 1) : -1;
      double2 pn_ = zero2, xn_ = zero2, qn_ = zero2;
      if (kn >= 0) {
        pn_ = p2[kn];
        if (xupd) xn_ = x2[kn];
        if (xupd && xmode == 2) qn_ = pp2[kn];
      }
      if (kc >= 0) dir_step(j, kc, pc, xc, qc);
      kc = kn;
      pc = pn_;
      xc = xn_;
      qc = qn_;
    }
  } else {
    for (int j0 = nj - 1; j0 >= 0; j0 -= ST_U2) {
      int k[ST_U2];
      double2 pv[ST_U2], xv[ST_U2], qv[ST_U2];
#pragma unroll
      for (int u = 0; u < ST_U2; ++u) {
        const int j = j0 - u;
        k[u] = j >= 0 ? pair_at(j) : -1;
        if (k[u] < 0) continue;
        pv[u] = p2[k[u]];
        xv[u] = xupd ? x2[k[u]] : pv[u];
        qv[u] = (xupd && xmode == 2) ? pp2[k[u]] : pv[u];
      }
#pragma unroll
      for (int u = 0; u < ST_U2; ++u)
        if (k[u] >= 0) dir_step(j0 - u, k[u], pv[u], xv[u], qv[u]);
    }
  }
  if (ts) g_step_ts[3][blockIdx.x] = gtimer();
  // this CTA's vector writes are done: the next operator kernel may launch
  // onto the SMs freed by the CTAs that finish first (it issues its first
  // factor copy and waits in griddepcontrol.wait for this grid to complete)
  pdl_trigger();
  const double sc = block_sum<ST_NT>(cc, scratch);
  if (threadIdx.x == 0) part[2 * G + blockIdx.x] = sc;
  if (!pcg_last_cta(&st->counter[2])) return;
  const double tc = pcg_sum_partials<ST_NT>(part + 2 * G, G, scratch);
  if (threadIdx.x == 0) {
    st->counter[2] = 0;
    st->pap = pap;
    st->alpha = alpha;
    st->red[1] = trr;
    st->red[2] = trz;
    if (stop) {
      if (bad) {
        st->error = PCG_ERR_RESID;
      } else {
        st->it = it;
        st->res = res;
        hist[it] = res;
        if (conv) st->converged = 1;
      }
      st->stop = 1;
      return;
    }
    st->red[3] = tc;
    st->it = it;
    st->res = res;
    hist[it] = res;
    if (conv) st->converged = 1;
    st->beta = beta;
    st->rho = trz;
    st->alpha_prev = alpha;
  }
}

// y = x on constrained rows, 0 elsewhere: the RED target of an operator apply
// (operator.cpp:87-90,141-143).  With an owner mask only the owner presets
// (a following interface sum-exchange then leaves exactly x).
__global__ void __launch_bounds__(VT)
    init_y_kernel(int64_t n_L, int m, const double* __restrict__ x, double* __restrict__ y,
                  const uint32_t* cons_mask, const uint32_t* own) {
  const int64_t stride = (int64_t)gridDim.x * VT;
  for (int c = 0; c < m; ++c)
    for (int64_t node = (int64_t)blockIdx.x * VT + threadIdx.x; node < n_L; node += stride) {
      const int64_t i = c * n_L + node;
      y[i] = (is_cons(cons_mask, node) && owned_w(own, node) != 0.0) ? x[i] : 0.0;
    }
}

// ------------------------------------------------------------------ host side
int vec_grid() { return capped_grid(int64_t(num_sms()) * 4, num_sms() * 4); }

namespace {
bool aligned16(const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}  // namespace

cudaError_t launch_init_y(cudaStream_t s, int64_t n_L, int m, const double* x, double* y,
                          const uint32_t* mask, const uint32_t* own) {
  if (!mask) return cudaMemsetAsync(y, 0, sizeof(double) * n_L * m, s);
  init_y_kernel<<<vec_grid(), VT, 0, s>>>(n_L, m, x, y, mask, own);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_init(cudaStream_t s, PcgState* st, int64_t n_L, int m, const double* b,
                            const double* d, double* dinv, double* x, double* r, double* p,
                            double* Ap, const uint32_t* mask, const uint32_t* own, double* part) {
  pcg_init_kernel<<<vec_grid(), VT, 0, s>>>(st, n_L, m, b, d, dinv, x, r, p, Ap, mask, own, part);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_init_finalize(cudaStream_t s, PcgState* st, double* hist) {
  pcg_init_finalize<<<1, 32, 0, s>>>(st, hist);
  count_launch();
  return cudaGetLastError();
}

cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int it, int64_t n_L, int m,
                              const double* d, double* r, const double* Ap, const uint32_t* own,
                              double* part, int rev) {
  const bool vec = (n_L % 2) == 0 && aligned16(d) && aligned16(r) && aligned16(Ap);
  auto k = vec ? (own ? pcg_update_kernel<true, true> : pcg_update_kernel<true, false>)
               : (own ? pcg_update_kernel<false, true> : pcg_update_kernel<false, false>);
  const cudaError_t err =
      launch_pdl(k, dim3(vec_grid()), dim3(VT), 0, s, st, it, n_L, m, d, r, Ap, own, part, rev);
  count_launch();
  return err;
}

cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int it, double* hist, int64_t n_L,
                                 int m, const double* d, const double* r, double* x, const double* p,
                                 const double* pprev, double* pout, double* Ap,
                                 const uint32_t* mask, const uint32_t* own, double* part, int rev,
                                 int xmode) {
  const bool vec = (n_L % 2) == 0 && aligned16(d) && aligned16(r) && aligned16(x) &&
                   aligned16(p) && aligned16(pprev) && aligned16(pout) && aligned16(Ap);
  auto k = vec ? pcg_direction_kernel<true> : pcg_direction_kernel<false>;
  const cudaError_t err = launch_pdl(k, dim3(vec_grid()), dim3(VT), 0, s, st, it, hist, n_L, m, d,
                                     r, x, p, pprev, pout, Ap, mask, own, part, rev, xmode);
  count_launch();
  return err;
}

}  // namespace hxf

namespace hxf {

int pcg_step_grid() { return num_sms(); }

// measurement only: per-CTA phase timestamps of the next fused step launches
void pcg_step_timestamps(int on, unsigned long long* out /* 4 x 1024, or nullptr */) {
  cudaMemcpyToSymbol(g_step_ts_on, &on, sizeof on);
  if (out) cudaMemcpyFromSymbol(out, g_step_ts, sizeof(unsigned long long) * 4 * 1024);
}

bool pcg_step_fusable(int64_t n_L, const double* d, const double* r, double* x, const double* p,
                      const double* pprev, double* pout, double* Ap) {
  static const bool off = [] {
    const char* v = std::getenv("HXF_PCG_FUSED");
    return v && v[0] == '0';
  }();
  static const bool coop = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, dev);
    return v != 0;
  }();
  return !off && coop && grid_cap() == 0 && (n_L % 2) == 0 && n_L * 3 < (int64_t(1) << 31) && aligned16(d) && aligned16(r) &&
         aligned16(x) && aligned16(p) && aligned16(pprev) && aligned16(pout) && aligned16(Ap);
}

cudaError_t pcg_launch_step(cudaStream_t s, PcgState* st, int it, double* hist, int64_t n_L, int m,
                            const double* d, double* r, double* x, const double* p,
                            const double* pprev, double* pout, double* Ap, const uint32_t* mask,
                            double* part, int rev, int xmode, bool ap_zero) {
  // (measured, C3 CG iteration: phase 1 / 2 unrolled 1/2 158.6 us, 2/2 158.1,
  // 1/4 178.3 (spills) vs 1/1 156.8 — kept 1/1)
  // evict-first stores: 0 none, 1 x and r (measured: C3 CG iteration 156.7 ->
  // 155.9 us), 2 + p, 3 + the Ap preset (both slower; so are write-through
  // st.global.wt stores of x and r: 153.7 -> 156.7 us)
  static const int cs = [] {
    const char* v = std::getenv("HXF_STEP_CS");
    return v ? std::atoi(v) : 1;
  }();
  static const bool pf = [] {  // HXF_STEP_PF=0: phase 2 without the one-step-ahead loads
    const char* v = std::getenv("HXF_STEP_PF");
    return !(v && v[0] == '0');
  }();
  auto kern = pf        ? pcg_step_kernel<1, 0, 1>
              : cs == 0 ? pcg_step_kernel<1, 1, 0>
              : cs == 2 ? pcg_step_kernel<1, 1, 2>
              : cs == 3 ? pcg_step_kernel<1, 1, 3>
                        : pcg_step_kernel<1, 1, 1>;
  static const cudaError_t attr =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM);
  if (attr != cudaSuccess) return attr;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pcg_step_grid());
  cfg.blockDim = dim3(ST_NT);
  cfg.dynamicSmemBytes = ST_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (grid barrier)
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, kern, st, it, hist, n_L, m, d, r, x,
                                             p, pprev, pout, Ap, mask, part, rev, xmode,
                                             ap_zero ? 1 : 0);
  count_launch();
  return err;
}

}  // namespace hxf
