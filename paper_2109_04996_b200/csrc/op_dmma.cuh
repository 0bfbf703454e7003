// K1 (collocated BP5/BP6, p = 7): fused operator on the FP64 tensor cores.
//   y = G^T D^T S D G x,  every 1-D contraction an 8x8x8 matrix product.
//
// The pencil kernel (op_pencil.cuh) is issue-bound: with all memory traffic
// ablated it still takes ~90 us at C3 (2400 warp-instructions per element).
// Here each 1-D contraction of an 8x8 slice is two DMMA m8n8k4 (FP64 tensor
// core, mma.sync) instructions instead of 64 DFMA lanes-worth, cutting the
// instruction count per element ~4x; the arithmetic (and its FP64 rounding
// model: fused multiply-adds) is unchanged.
//
// One element per CTA of NW warps (4 by default, KK = 8/NW planes each); lane
// l: g = l>>2, t = l&3 (the mma fragment coordinates).  "dist X": a lane owns
// points (k, j = g, i = 2t..2t+1) of the warp's planes k in {KK w .. KK w +
// KK-1}; "dist Z": (k = g, j, i = 2t..2t+1) for the warp's rows j in the same
// range.
//   x-dir  G0_k = U_k D^T    (M = j, N = o, K = a)  -> dist X, registers
//   y-dir  G1_k = D U_k      (M = o, N = i, K = b)  -> dist X, registers
//   z-dir  G2_j = D U_(.j.)  (M = o, N = i, K = c)  -> dist Z -> slab Z
//   QFunction on dist X (factors from the TMA-staged slab), V0 -> A, V1 -> B,
//   V2 -> Z;  x^T and y^T accumulate into one fragment (dist X), z^T lands in
//   dist Z and is transposed through slab B before the FP64 RED scatter.
// The only D operands a lane ever needs are D[g][4ks+t] and D[4ks+t][g]
// (4 registers).  Slabs are [k][R][col] with R = j ^ (k & 1) and the 16-byte
// half of each row flipped by bit 1 of R, which keeps every fragment load at
// its 2-wavefront minimum and every dist-X / dist-Z pair access at 4.
// Gather software-pipelined (next item's z-lines in registers), geometric
// factors by one bulk async copy (TMA engine, L2 evict_first) per element,
// issued as soon as the previous element's QFunction consumed them.
// Reference semantics: proj/src/operator.cpp:64-144 (see op_kernel.cuh).
#pragma once
// CTAs per SM the register budget targets (measured: 5 -> 96 registers, no spills,
// but 2.5 % slower at C3 and 9 % at C4 p=7 than 4 -> 128 registers)
#ifndef HXF_DMMA_MINB3
#define HXF_DMMA_MINB3 4
#endif
#ifndef HXF_DMMA_TMA_NB  // TMA x slabs per CTA: 2 = issued two work items ahead, 1 = one
#define HXF_DMMA_TMA_NB 2
#endif
#ifndef HXF_DMMA_TMA_MINB  // CTAs per SM the TMA variant's register budget targets
#define HXF_DMMA_TMA_MINB 4
#endif
#ifndef HXF_DMMA_QPF  // elements of geometric factors prefetched into L2 beyond the staged one
#define HXF_DMMA_QPF 0
#endif
#ifndef HXF_DMMA_MINB
#define HXF_DMMA_MINB 4
#endif
#include <cuda.h>  // CUtensorMap (type only; encoded through the runtime's driver entry point)

#include "hxf_device.cuh"
#include "hxf_internal.h"
#include "pcg_device.cuh"

namespace hxf {

template <int NC_, int GM_, int NW_ = 4, int NP_ = 8, int NS_ = 1, bool TMA_ = false>
struct DmmaTraits {
  // TMA: the element's x slab arrives by one tensor-map copy
  // (cp.async.bulk.tensor.4d over the [m][NZ][NY][NX] lattice, double-
  // buffered two work items ahead) instead of per-lane loads; structured box
  // only (GM = 0), lattice rows 16-byte multiples.  A box must start on a
  // 16-byte boundary (an odd f64 column faults: tools/micro/drv), so the box
  // is 12 columns wide from the even column at or below the element's first
  // and the element sits at column offset o = ix0 & 1; 12-double rows keep the
  // x- and y-direction fragment loads at their 2-wavefront minimum (z: 4)
  static constexpr bool TMA = TMA_;
  static_assert(!TMA_ || GM_ == 0, "TMA gather needs the structured box");
  // NS stages of staged geometric factors (1: refill right after the
  // QFunction consumed them; 2: two elements in flight per CTA)
  static constexpr int NS = NS_;
  // NW warps per element; warp w owns planes / rows KK w .. KK w + KK-1
  static constexpr int P = 8, NC = NC_, GM = GM_, P3 = 512, NW = NW_, NT = 32 * NW_, KK = 8 / NW_;
  // NP = p+1 nodes per direction: 8, or 5..7 zero-padded to the 8^3 tile
  // (padded rows / columns of D are 0, padded points masked like constrained
  // ones; the geometric factors stay compact, NP^3 per plane)
  static constexpr int NP = NP_, NP3 = NP_ * NP_ * NP_;
  static constexpr bool PAD = NP_ < 8;
  static_assert(NP_ >= 5 && NP_ <= 8, "DMMA tile holds 5..8 nodes per direction");
  static_assert(NW_ == 2 || NW_ == 4 || NW_ == 8, "8 planes split over NW warps");
  // CTAs per SM the register budget is sized for (tuned at C3: NW = 4 -> 122
  // registers, 4 CTAs; NW = 2 needs 224 registers to keep its loads in flight)
  static constexpr int MINB = NW_ == 8 ? 3
                              : TMA_   ? HXF_DMMA_TMA_MINB
                                       : (NC_ == 3 ? HXF_DMMA_MINB3 : HXF_DMMA_MINB);
  static constexpr int SLAB = 512;   // doubles
  static constexpr int QDS = 6 * NP3;
  // TMA x buffers first (a TMA destination must be 128-byte aligned)
  static constexpr int XW = 12, XSLAB = XW * 64;  // box {12, 8, 8, 1}: 6 KB
  static constexpr int XNB = HXF_DMMA_TMA_NB;
  static constexpr int OFF_X = 0;
  static constexpr int XBUF = TMA_ ? XNB * XSLAB : 0;
  static constexpr int OFF_QD = OFF_X + XBUF;
  static constexpr int OFF_A = OFF_QD + NS_ * QDS;  // U, then V0
  static constexpr int OFF_B = OFF_A + SLAB;  // V1, then Y2 (dist-Z -> dist-X transpose)
  static constexpr int OFF_Z = OFF_B + SLAB;  // G2, then V2
  static constexpr int SMEM_BYTES = (OFF_Z + SLAB) * 8;

  __device__ static __forceinline__ int off(int k, int j, int i) {
    const int R = j ^ (k & 1);
    return k * 64 + R * 8 + (i ^ (((R >> 1) & 1) << 2));
  }
  // element point (k, j, i) in a TMA slab whose columns start o before it
  __device__ static __forceinline__ int tix(int k, int j, int i, int o) {
    return (k * 8 + j) * XW + o + i;
  }
};

// One tensor-map box copy global -> shared (4-D coordinates, innermost
// first), completion counted on `bar`.
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            int c, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(c), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <class T>
__global__ void __launch_bounds__(T::NT, T::MINB)
    op_dmma_kernel(const __grid_constant__ OpParams prm, const __grid_constant__ CUtensorMap xmap) {
  constexpr int NC = T::NC, P3 = T::P3, NT = T::NT, KK = T::KK;
  extern __shared__ __align__(128) double dmma_smem[];
  double* smem = dmma_smem;
  __shared__ __align__(8) uint64_t qbars[T::NS];
  __shared__ __align__(8) uint64_t xbars[2];
  __shared__ double red_scratch[NT / 32 + 1];
  double* sX = smem + T::OFF_X;  // TMA: two x slabs (work items q, q+1 / q+2)

  // measurement-only ablation (HXF_ABLATE bit 16): memory traffic and barriers
  // without the contractions / QFunction arithmetic
  const bool skipc = (prm.ablate & 16) != 0;
  const int tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31, g = l >> 2, t = l & 3;
  double* sQD = smem + T::OFF_QD;
  double* SA = smem + T::OFF_A;
  double* SB = smem + T::OFF_B;
  double* SZ = smem + T::OFF_Z;

  // the only D entries this lane ever multiplies by (fragment coordinates)
  double Dr[2], Dc[2];
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    constexpr int NP = T::NP;
    const bool in = g < NP && ks * 4 + t < NP;
    Dr[ks] = in ? __ldg(prm.D + g * NP + ks * 4 + t) : 0.0;    // D[g][4ks+t]
    Dc[ks] = in ? __ldg(prm.D + (ks * 4 + t) * NP + g) : 0.0;  // D[4ks+t][g]
  }

  const int64_t nsteps = prm.E;
  const int64_t G = gridDim.x;
  const int64_t NXY = prm.NX * prm.NY;
  uint64_t policy = 0;
  // sweep position -> element: last to first when prm.rev (the CG driver
  // alternates sweep directions so each kernel starts where the previous one's
  // most recent, L2-resident, vector traffic is)
  auto elem = [&](int64_t s) {
    const int64_t k = prm.rev ? nsteps - 1 - s : s;
    return prm.elist ? (int64_t)__ldg(prm.elist + k) : k;  // subset (partition overlap)
  };
  // sweep step s of this CTA goes to stage (s / G) % NS
  auto issue_qdata = [&](int64_t e, int stage) {
    mbar_arrive_expect_tx(&qbars[stage], (uint32_t)(T::QDS * 8));
    bulk_g2s(sQD + stage * T::QDS, prm.qd + elem(e) * T::QDS, (uint32_t)(T::QDS * 8), &qbars[stage],
             policy);
  };
  // the first element's factors do not depend on the previous kernel: request
  // them before the PDL wait so the copy overlaps that kernel's tail
  const bool first_qd = (int64_t)blockIdx.x < nsteps && !(prm.ablate & 4);
  if (tid == 0) {
    for (int i = 0; i < T::NS; ++i) mbar_init(&qbars[i], 1);
    if constexpr (T::TMA) {
      if (smem_u32(sX) & 127u) __trap();  // TMA destinations are 128-byte aligned
      mbar_init(&xbars[0], 1);
      mbar_init(&xbars[1], 1);
    }
    fence_mbar_init();
    policy = l2_evict_first_policy();
    if (first_qd) {
      issue_qdata(blockIdx.x, 0);
      for (int d = 1; d <= HXF_DMMA_QPF; ++d)
        if ((int64_t)blockIdx.x + (T::NS - 1 + d) * G < nsteps)
          bulk_prefetch_l2(prm.qd + elem(blockIdx.x + (T::NS - 1 + d) * G) * T::QDS,
                           (uint32_t)(T::QDS * 8));
      if (T::NS > 1 && (int64_t)blockIdx.x + G < nsteps) issue_qdata(blockIdx.x + G, 1);
    }
  }
  pdl_wait();     // x, y, stop and the PCG state come from the previous kernels
  // (no early trigger: dependents launch when this grid completes)
  if (prm.stop && *prm.stop) {
    if (tid == 0 && first_qd) {  // no copy in flight at exit
      mbar_wait(&qbars[0], 0);
      if (T::NS > 1 && (int64_t)blockIdx.x + G < nsteps) mbar_wait(&qbars[1], 0);
    }
    return;
  }

  // Gather geometry of one element for this lane: node of (i = 2t, j = g,
  // k = 4w) and constraint bits (bit 2*kk + h: node (i = 2t + h, k = 4w + kk)).
  struct Geo {
    int64_t key;
    uint32_t cmask;
    bool active;
    int ix0, iy0, iz0;  // element origin on the lattice (TMA box coordinates)
  };
  auto node_of = [&](const Geo& q, int kk, int h) -> int64_t {
    if constexpr (T::GM == 0) return q.key + (int64_t)kk * NXY + h;
    if (prm.idx)
      return (int64_t)prm.idx[q.key * T::NP3 + (2 * t + h) + T::NP * (g + T::NP * (KK * w + kk))];
    return q.key + (int64_t)kk * NXY + h;
  };
  // loop-invariant lane masks: which of this lane's points lie on each of the
  // six faces of an element (bit 2*kk + h: point i = 2t+h, j = g, k = KK w + kk)
  uint32_t fmask[6] = {0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
  for (int kk = 0; kk < KK; ++kk)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * t + h, k = KK * w + kk;
      const uint32_t bit = 1u << (2 * kk + h);
      fmask[0] |= i == 0 ? bit : 0u;
      fmask[1] |= i == T::NP - 1 ? bit : 0u;
      fmask[2] |= g == 0 ? bit : 0u;
      fmask[3] |= g == T::NP - 1 ? bit : 0u;
      fmask[4] |= k == 0 ? bit : 0u;
      fmask[5] |= k == T::NP - 1 ? bit : 0u;
    }
  const FastDiv divx((uint32_t)prm.nx), divy((uint32_t)prm.ny);
  auto geometry = [&](int64_t s) {
    Geo q{};
    q.active = s < nsteps;
    if (!q.active) return q;
    const int64_t e = elem(s);
    if (T::GM == 1 && prm.idx) {
      q.key = e;
    } else {
      // element lattice position (E < 2^31: 32-bit fast division)
      const uint32_t e32 = (uint32_t)e, r = divx.div(e32), ez = divy.div(r);
      const uint32_t ex = e32 - r * (uint32_t)prm.nx, ey = r - ez * (uint32_t)prm.ny;
      const int64_t ix0 = (int64_t)ex * (T::NP - 1), iy0 = (int64_t)ey * (T::NP - 1),
                    iz0 = (int64_t)ez * (T::NP - 1);
      q.ix0 = (int)ix0;
      q.iy0 = (int)iy0;
      q.iz0 = (int)iz0;
      q.key = (ix0 + 2 * t) + prm.NX * (iy0 + g) + NXY * (iz0 + KK * w);
      if (T::GM == 0 && prm.cons_mode == 1) {
        // on_bnd_face per point, as element-face flags x lane masks
        const int f = prm.bnd_faces;
        uint32_t cm = 0u;
        if ((f & 1) && ix0 == 0) cm |= fmask[0];
        if ((f & 2) && ix0 + T::NP - 1 == prm.NX - 1) cm |= fmask[1];
        if ((f & 4) && iy0 == 0) cm |= fmask[2];
        if ((f & 8) && iy0 + T::NP - 1 == prm.NY - 1) cm |= fmask[3];
        if ((f & 16) && iz0 == 0) cm |= fmask[4];
        if ((f & 32) && iz0 + T::NP - 1 == prm.NZ - 1) cm |= fmask[5];
        q.cmask = cm;
      }
    }
    if constexpr (T::PAD) {
      // padding points of the 8^3 tile: masked like constrained nodes
#pragma unroll
      for (int kk = 0; kk < KK; ++kk)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (2 * t + h >= T::NP || g >= T::NP || KK * w + kk >= T::NP) q.cmask |= 1u << (2 * kk + h);
    }
    if (T::GM == 1 && prm.cons_mode == 2) {
#pragma unroll
      for (int kk = 0; kk < KK; ++kk)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (T::PAD && ((q.cmask >> (2 * kk + h)) & 1u)) continue;
          const int64_t node = node_of(q, kk, h);
          q.cmask |= ((prm.cons_mask[node >> 5] >> (node & 31)) & 1u) << (2 * kk + h);
        }
    }
    return q;
  };
  auto load_lines = [&](const Geo& q, int c, double* xn) {
    const double* xc = prm.x + c * prm.n_L;
    // structured box: a lane's node pair (i = 2t, 2t+1) is 16-byte aligned iff
    // its first node is even (uniform across the element when NX, n_L even)
    if (T::GM == 0 && !T::PAD && q.active && !(prm.ablate & 1) && ((reinterpret_cast<uintptr_t>(xc) +
                                                         8 * q.key) & 15u) == 0 &&
        (prm.NX & 1) == 0) {
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(xc + node_of(q, kk, 0)));
        xn[2 * kk] = v.x;
        xn[2 * kk + 1] = v.y;
      }
      return;
    }
#pragma unroll
    for (int kk = 0; kk < KK; ++kk)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        xn[2 * kk + h] = (q.active && !(prm.ablate & 1) && !(T::PAD && ((q.cmask >> (2 * kk + h)) & 1u)))
                             ? __ldg(xc + node_of(q, kk, h))
                             : 1.0;
  };

  // constrained rows of a work item: y = x (operator.cpp:87-90,141-143), plain
  // stores of the raw gathered values (idempotent across elements sharing a node)
  auto store_cons = [&](const Geo& gq, int c, const double* raw) {
    if (T::PAD || !prm.cons_store || !gq.active || gq.cmask == 0) return;
    double* yc = prm.y + c * prm.n_L;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if ((gq.cmask >> (2 * kk + h)) & 1u) yc[node_of(gq, kk, h)] = raw[2 * kk + h];
  };

  Geo gcur = geometry(blockIdx.x);
  Geo gpf = NC > 1 ? gcur : geometry(blockIdx.x + G);
  // TMA: work item q's slab lands in sX[q & 1], issued two items ahead
  auto issue_x = [&](const Geo& gq, int c, int buf) {
    mbar_arrive_expect_tx(&xbars[buf], (uint32_t)(T::XSLAB * 8));
    tma_load_4d(sX + buf * T::XSLAB, &xmap, gq.ix0 & ~1, gq.iy0, gq.iz0, c, &xbars[buf]);
  };
  double xn[2 * KK];
  double u[2 * KK];
  if constexpr (T::TMA) {
    if (tid == 0) {
      if (gcur.active) issue_x(gcur, 0, 0);
      if (T::XNB == 2 && gpf.active) issue_x(gpf, 1 % NC, 1);
    }
  } else {
    load_lines(gcur, 0, xn);
#pragma unroll
    for (int m = 0; m < 2 * KK; ++m) u[m] = (gcur.active && !((gcur.cmask >> m) & 1u)) ? xn[m] : 0.0;
    store_cons(gcur, 0, xn);
    load_lines(gpf, 1 % NC, xn);
  }
  __syncthreads();  // mbarrier init visible

  double dot_acc = 0.0;
  int it = 0, q = 0;
  Geo gnext_el{};
#pragma unroll 1
  for (int64_t e = blockIdx.x; e < nsteps; e += G, ++it) {
#pragma unroll 1
    for (int c = 0; c < NC; ++c, ++q) {
      double* yc = prm.y + c * prm.n_L;
      double* X = sX + (q % T::XNB) * T::XSLAB;  // TMA: this item's slab
      const int xo = gcur.ix0 & 1;          // TMA: the element's column offset in it
      Geo gnext{};                          // TMA: item q+2 (its slab is issued after (B))
      const Geo gi1 = gpf;                  // TMA: item q+1 (single-slab variant)
      if constexpr (T::TMA) {
        // ---- G: the slab is in shared memory; zero the constrained (and
        // padding) points in place, storing y = x there first (single apply) ----
        if (c == NC - 1) gnext_el = gpf;
        gnext = ((q + 2) / NC == (q + 1) / NC && NC > 1)
                    ? gpf
                    : geometry((int64_t)blockIdx.x + (int64_t)((q + 2) / NC) * G);
        mbar_wait(&xbars[q % T::XNB], (uint32_t)((q / T::XNB) & 1));
        if (gcur.cmask) {
#pragma unroll
          for (int kk = 0; kk < KK; ++kk)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if ((gcur.cmask >> (2 * kk + h)) & 1u) {
                double* px = X + T::tix(KK * w + kk, g, 2 * t + h, xo);
                if (!T::PAD && prm.cons_store) yc[node_of(gcur, kk, h)] = *px;
                *px = 0.0;
              }
        }
        gpf = gnext;
      } else {
        // ---- G: this lane's masked dist-X pairs into slab A ----
#pragma unroll
        for (int kk = 0; kk < KK; ++kk)
          *reinterpret_cast<double2*>(SA + T::off(KK * w + kk, g, 2 * t)) =
              make_double2(u[2 * kk], u[2 * kk + 1]);
        // next item's raw lines: land while this item computes
        if (c == NC - 1) gnext_el = gpf;  // item q+1 starts the next element
        const Geo gn = ((q + 2) / NC == (q + 1) / NC && NC > 1)
                           ? gpf
                           : geometry((int64_t)blockIdx.x + (int64_t)((q + 2) / NC) * G);
        double nx_[2 * KK];
#pragma unroll
        for (int m = 0; m < 2 * KK; ++m) nx_[m] = xn[m];
        // masked values of item q+1 are formed when it starts (gpf)
        load_lines(gn, (q + 2) % NC, xn);
        store_cons(gpf, (q + 1) % NC, nx_);
#pragma unroll
        for (int m = 0; m < 2 * KK; ++m)
          u[m] = (gpf.active && !((gpf.cmask >> m) & 1u)) ? nx_[m] : 0.0;  // item q+1
        gpf = gn;
      }
      // forward operand: the TMA slab (swizzled) or slab A
      auto U = [&](int k, int j, int i) -> double {
        if constexpr (T::TMA) return X[T::tix(k, j, i, xo)];
        return SA[T::off(k, j, i)];
      };
      __syncthreads();  // (A) slab A complete

      // ---- forward contractions ----
      double g0[KK][2], g1[KK][2];
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        const int k = KK * w + kk;
        double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          if (!skipc) dmma(c0, c1, U(k, g, 4 * ks + t), Dr[ks]);  // x: U_k[j][a] . D^T[a][o]
          if (!skipc) dmma(d0, d1, Dr[ks], U(k, 4 * ks + t, g));  // y: D[o][b] . U_k[b][i]
        }
        g0[kk][0] = c0;
        g0[kk][1] = c1;
        g1[kk][0] = d0;
        g1[kk][1] = d1;
      }
#pragma unroll
      for (int jj = 0; jj < KK; ++jj) {
        const int j = KK * w + jj;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) if (!skipc) dmma(c0, c1, Dr[ks], U(4 * ks + t, j, g));
        *reinterpret_cast<double2*>(SZ + T::off(g, j, 2 * t)) = make_double2(c0, c1);  // dist Z
      }
      const int stg = T::NS > 1 ? (it & 1) : 0;
      const double* sQDs = sQD + stg * T::QDS;
      if (c == 0 && !(prm.ablate & 4)) mbar_wait(&qbars[stg], (uint32_t)((it / T::NS) & 1));
      if constexpr (T::TMA) fence_proxy_async_smem();  // generic accesses of X before its refill
      __syncthreads();  // (B) G2 complete, slab A (TMA: this item's x slab) free
      if constexpr (T::TMA) {
        if (T::XNB == 2 && tid == 0 && gnext.active) issue_x(gnext, (q + 2) % NC, q & 1);
        if (T::XNB == 1 && tid == 0 && gi1.active) issue_x(gi1, (q + 1) % NC, 0);
      }

      // ---- QFunction on dist X (qfunction.cpp:135-162) ----
      double energy = 0.0;
#pragma unroll
      for (int kk = 0; kk < KK && !skipc; ++kk) {
        const int k = KK * w + kk;
        const int sp = T::off(k, g, 2 * t);
        const double2 z2 = *reinterpret_cast<const double2*>(SZ + sp);
        double2 s[6];
        if constexpr (!T::PAD) {
          const int pt = k * 64 + g * 8 + 2 * t;
#pragma unroll
          for (int m = 0; m < 6; ++m) s[m] = *reinterpret_cast<const double2*>(sQDs + m * P3 + pt);
        } else {
          // compact NP^3 factors; padding points get 0 (their V is then 0)
          constexpr int NP = T::NP;
          const int pt = (k * NP + g) * NP + 2 * t;
          const bool v0 = k < NP && g < NP && 2 * t < NP, v1 = k < NP && g < NP && 2 * t + 1 < NP;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            s[m].x = v0 ? sQDs[m * T::NP3 + pt] : 0.0;
            s[m].y = v1 ? sQDs[m * T::NP3 + pt + 1] : 0.0;
          }
        }
        double v0[2], v1[2], v2[2];
        const double gz[2] = {z2.x, z2.y};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double a0 = g0[kk][h], a1 = g1[kk][h], a2 = gz[h];
          const double s00 = h ? s[0].y : s[0].x, s01 = h ? s[1].y : s[1].x;
          const double s02 = h ? s[2].y : s[2].x, s11 = h ? s[3].y : s[3].x;
          const double s12 = h ? s[4].y : s[4].x, s22 = h ? s[5].y : s[5].x;
          v0[h] = s00 * a0 + s01 * a1 + s02 * a2;
          v1[h] = s01 * a0 + s11 * a1 + s12 * a2;
          v2[h] = s02 * a0 + s12 * a1 + s22 * a2;
          // p.(A p) over free nodes = sum_points grad u . S grad u
          energy += a0 * v0[h] + a1 * v1[h] + a2 * v2[h];
        }
        *reinterpret_cast<double2*>(SA + sp) = make_double2(v0[0], v0[1]);
        *reinterpret_cast<double2*>(SB + sp) = make_double2(v1[0], v1[1]);
        *reinterpret_cast<double2*>(SZ + sp) = make_double2(v2[0], v2[1]);
      }
      dot_acc += prm.coef * energy;
      if (c == NC - 1) fence_proxy_async_smem();  // generic reads of the factors before the refill
      __syncthreads();  // (C) V0, V1, V2 complete
      if (c == NC - 1 && tid == 0 && e + T::NS * G < nsteps && !(prm.ablate & 4))
      {
        issue_qdata(e + T::NS * G, stg);
        // keep DRAM busy one element further ahead: the staged copy of that
        // element then hits L2
        const int64_t pf = e + (T::NS + HXF_DMMA_QPF) * G;
        if (HXF_DMMA_QPF > 0 && pf < nsteps)
          bulk_prefetch_l2(prm.qd + elem(pf) * T::QDS, (uint32_t)(T::QDS * 8));
      }

      // ---- transposed contractions ----
      double y01[KK][2];
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        const int k = KK * w + kk;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          if (!skipc) dmma(c0, c1, SA[T::off(k, g, 4 * ks + t)], Dc[ks]);  // x^T: V0_k[j][a] . D[a][i]
          if (!skipc) dmma(c0, c1, Dc[ks], SB[T::off(k, 4 * ks + t, g)]);  // y^T: D^T[j][b] . V1_k[b][i]
        }
        y01[kk][0] = c0;
        y01[kk][1] = c1;
      }
      double y2z[KK][2];
#pragma unroll
      for (int jj = 0; jj < KK; ++jj) {
        const int j = KK * w + jj;
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) if (!skipc) dmma(c0, c1, Dc[ks], SZ[T::off(4 * ks + t, j, g)]);  // z^T
        y2z[jj][0] = c0;
        y2z[jj][1] = c1;
      }
      __syncthreads();  // (D) slab B (V1) free
#pragma unroll
      for (int jj = 0; jj < KK; ++jj)
        *reinterpret_cast<double2*>(SB + T::off(g, KK * w + jj, 2 * t)) =
            make_double2(y2z[jj][0], y2z[jj][1]);
      __syncthreads();  // (E) Y2 in slab B (dist Z)

      // ---- combine on dist X, G^T scatter (constrained rows preset by the caller) ----
      if (gcur.active) {
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
          const double2 z2 = *reinterpret_cast<const double2*>(SB + T::off(KK * w + kk, g, 2 * t));
          const double yk0 = prm.coef * (y01[kk][0] + z2.x);
          const double yk1 = prm.coef * (y01[kk][1] + z2.y);
          if (!(prm.ablate & 2)) {
            red_add_if(yc + node_of(gcur, kk, 0), yk0, !((gcur.cmask >> (2 * kk)) & 1u));
            red_add_if(yc + node_of(gcur, kk, 1), yk1, !((gcur.cmask >> (2 * kk + 1)) & 1u));
          }
        }
      }
      __syncthreads();  // (F) slab B free for the next item
    }
    gcur = gnext_el;  // == geometry(e + G), computed one item ahead
  }

  if (prm.dot_partials) {
    const double s = block_sum<NT>(dot_acc, red_scratch);
    if (tid == 0) prm.dot_partials[blockIdx.x] = s;
    pcg_alpha_epilogue<NT>(prm.fin, red_scratch);
  }
}

}  // namespace hxf
