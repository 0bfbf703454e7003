// K1 (collocated BP6, p = 6, 7): three-component fused operator on the FP64
// tensor cores with the components batched through every phase.
//   y_c = G^T D^T S D G x_c,  c = 0, 1, 2 (the same S for every component)
//
// op_dmma.cuh runs the three components of an element one after the other:
// 6 barriers each, the element's geometric factors re-read from shared memory
// three times, and per phase only one component's dependent chain of fragment
// loads -> DMMA per warp — latency-bound (BP6 C4 p = 7: issue-active 41 %,
// short-scoreboard stalls on shared memory, 0.49 of HBM).  Here each phase
// does all three components back to back (three independent chains per warp),
// the QFunction loads a point's six factors once for the three components,
// and an element costs 5 barriers instead of 18.
//
// One element per CTA of 8 warps (one plane / one row per warp: KK = 1), two
// CTAs per SM.  Lane l: g = l>>2, t = l&3.  "dist X": the lane owns points
// (k = w, j = g, i = 2t..2t+1) of every component; "dist Z": (k = g, j = w,
// i = 2t..2t+1).  Per component c the slabs A_c (U, then V0), B_c (V1, then
// the z^T transpose) and Z_c (G2, then V2) use op_dmma.cuh's swizzled layout;
// NP = 6, 7 (p = 5, 6) run on the zero-padded 8^3 tile as there.
//   G  masked dist-X pairs of the 3 components -> A_c (raw values loaded one
//      element ahead); the next element's loads issued        | barrier A
//   F  per c: x- and y-products (registers), z-product -> Z_c   | wait factors, B
//   Q  per point pair: 6 factors once; per c: V0 -> A_c, V1 -> B_c, V2 -> Z_c;
//      p.Ap as sum grad u . S grad u                            | C, refill factors
//   T  per c: x^T + y^T (registers, dist X), z^T (registers, dist Z)  | D
//      z^T -> B_c                                               | E
//   S  per c: combine on dist X, FP64 RED scatter
// Reference semantics: proj/src/operator.cpp:64-144 (see op_kernel.cuh).
#pragma once
#include "hxf_device.cuh"
#include "hxf_internal.h"
#include "op_dmma.cuh"  // dmma(), DmmaTraits::off (slab swizzle)
#include "pcg_device.cuh"

#ifndef HXF_DMMA3_MINB
#define HXF_DMMA3_MINB 2
#endif

namespace hxf {

template <int GM_, int NP_ = 8>
struct Dmma3Traits {
  static constexpr int NC = 3, GM = GM_, NW = 8, NT = 256, P3 = 512;
  static constexpr int NP = NP_, NP3 = NP_ * NP_ * NP_;
  static constexpr bool PAD = NP_ < 8;
  static_assert(NP_ >= 5 && NP_ <= 8, "DMMA tile holds 5..8 nodes per direction");
  static constexpr int MINB = HXF_DMMA3_MINB;
  static constexpr int SLAB = 512;
  static constexpr int QDS = 6 * NP3;
  static constexpr int OFF_QD = 0;
  static constexpr int OFF_A = OFF_QD + QDS;       // A_c at OFF_A + c * SLAB
  static constexpr int OFF_B = OFF_A + 3 * SLAB;   // B_c
  static constexpr int OFF_Z = OFF_B + 3 * SLAB;   // Z_c
  static constexpr int SMEM_BYTES = (OFF_Z + 3 * SLAB) * 8;
  __device__ static __forceinline__ int off(int k, int j, int i) {
    const int R = j ^ (k & 1);
    return k * 64 + R * 8 + (i ^ (((R >> 1) & 1) << 2));
  }
};

template <class T>
__global__ void __launch_bounds__(T::NT, T::MINB) op_dmma3_kernel(const __grid_constant__ OpParams prm) {
  constexpr int NT = T::NT, NP = T::NP;
  extern __shared__ __align__(128) double d3_smem[];
  __shared__ __align__(8) uint64_t qbar;
  __shared__ double red_scratch[NT / 32 + 1];
  double* sQD = d3_smem + T::OFF_QD;
  const int tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31, g = l >> 2, t = l & 3;
  auto SA = [&](int c) { return d3_smem + T::OFF_A + c * T::SLAB; };
  auto SB = [&](int c) { return d3_smem + T::OFF_B + c * T::SLAB; };
  auto SZ = [&](int c) { return d3_smem + T::OFF_Z + c * T::SLAB; };

  double Dr[2], Dc[2];  // D[g][4ks+t], D[4ks+t][g] (zero outside NP x NP)
#pragma unroll
  for (int ks = 0; ks < 2; ++ks) {
    const bool in = g < NP && ks * 4 + t < NP;
    Dr[ks] = in ? __ldg(prm.D + g * NP + ks * 4 + t) : 0.0;
    Dc[ks] = in ? __ldg(prm.D + (ks * 4 + t) * NP + g) : 0.0;
  }

  const int64_t nsteps = prm.E;
  const int64_t G = gridDim.x;
  const int64_t NXY = prm.NX * prm.NY;
  uint64_t policy = 0;
  auto elem = [&](int64_t s) {
    const int64_t k = prm.rev ? nsteps - 1 - s : s;
    return prm.elist ? (int64_t)__ldg(prm.elist + k) : k;
  };
  auto issue_qdata = [&](int64_t s) {
    mbar_arrive_expect_tx(&qbar, (uint32_t)(T::QDS * 8));
    bulk_g2s(sQD, prm.qd + elem(s) * T::QDS, (uint32_t)(T::QDS * 8), &qbar, policy);
  };
  const bool first_qd = (int64_t)blockIdx.x < nsteps && !(prm.ablate & 4);
  if (tid == 0) {
    mbar_init(&qbar, 1);
    fence_mbar_init();
    policy = l2_evict_first_policy();
    if (first_qd) issue_qdata(blockIdx.x);
  }
  pdl_wait();  // x, y, stop and the PCG state come from the previous kernels
  if (prm.stop && *prm.stop) {
    if (tid == 0 && first_qd) mbar_wait(&qbar, 0);  // no copy in flight at exit
    return;
  }

  // this lane's gather / scatter points of an element: (i = 2t + h, j = g, k = w)
  struct Geo {
    int64_t key;
    uint32_t cmask;  // bit h: point (2t + h, g, w) constrained (or padding)
    bool active;
  };
  auto node_of = [&](const Geo& q, int h) -> int64_t {
    if constexpr (T::GM == 0) return q.key + h;
    if (prm.idx) return (int64_t)prm.idx[q.key * T::NP3 + (2 * t + h) + NP * (g + NP * w)];
    return q.key + h;
  };
  const FastDiv divx((uint32_t)prm.nx), divy((uint32_t)prm.ny);
  auto geometry = [&](int64_t s) {
    Geo q{};
    q.active = s < nsteps;
    if (!q.active) return q;
    const int64_t e = elem(s);
    if (T::GM == 1 && prm.idx) {
      q.key = e;
    } else {
      const uint32_t e32 = (uint32_t)e, r = divx.div(e32), ez = divy.div(r);
      const uint32_t ex = e32 - r * (uint32_t)prm.nx, ey = r - ez * (uint32_t)prm.ny;
      const int64_t ix0 = (int64_t)ex * (NP - 1), iy0 = (int64_t)ey * (NP - 1), iz0 = (int64_t)ez * (NP - 1);
      q.key = (ix0 + 2 * t) + prm.NX * (iy0 + g) + NXY * (iz0 + w);
      if (T::GM == 0 && prm.cons_mode == 1) {
        const int f = prm.bnd_faces;
        uint32_t cm = 0u;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = 2 * t + h;
          const bool on = ((f & 1) && ix0 == 0 && i == 0) ||
                          ((f & 2) && ix0 + NP - 1 == prm.NX - 1 && i == NP - 1) ||
                          ((f & 4) && iy0 == 0 && g == 0) ||
                          ((f & 8) && iy0 + NP - 1 == prm.NY - 1 && g == NP - 1) ||
                          ((f & 16) && iz0 == 0 && w == 0) ||
                          ((f & 32) && iz0 + NP - 1 == prm.NZ - 1 && w == NP - 1);
          cm |= on ? (1u << h) : 0u;
        }
        q.cmask = cm;
      }
    }
    if constexpr (T::PAD) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (2 * t + h >= NP || g >= NP || w >= NP) q.cmask |= 1u << h;
    }
    if (T::GM == 1 && prm.cons_mode == 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (T::PAD && ((q.cmask >> h) & 1u)) continue;
        const int64_t node = node_of(q, h);
        q.cmask |= ((prm.cons_mask[node >> 5] >> (node & 31)) & 1u) << h;
      }
    }
    return q;
  };
  // raw x pairs of the three components (padding points read nothing)
  auto load_x = [&](const Geo& q, double* xn) {
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        xn[2 * c + h] = (q.active && !(prm.ablate & 1) && !(T::PAD && ((q.cmask >> h) & 1u)))
                            ? __ldg(prm.x + c * prm.n_L + node_of(q, h))
                            : 0.0;
  };

  Geo gcur = geometry(blockIdx.x);
  double xn[6];
  load_x(gcur, xn);
  __syncthreads();  // mbarrier init visible

  double dot_acc = 0.0;
  int it = 0;
#pragma unroll 1
  for (int64_t e = blockIdx.x; e < nsteps; e += G, ++it) {
    // ---- G: masked dist-X pairs -> A_c (y = x on constrained rows for a
    //      zero-filled single apply); the next element's raw pairs in flight ----
    {
      const int sp = T::off(w, g, 2 * t);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double u0 = ((gcur.cmask >> 0) & 1u) ? 0.0 : xn[2 * c];
        const double u1 = ((gcur.cmask >> 1) & 1u) ? 0.0 : xn[2 * c + 1];
        *reinterpret_cast<double2*>(SA(c) + sp) = make_double2(u0, u1);
        if (!T::PAD && prm.cons_store && gcur.cmask) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if ((gcur.cmask >> h) & 1u) prm.y[c * prm.n_L + node_of(gcur, h)] = xn[2 * c + h];
        }
      }
    }
    const Geo gnext = geometry(e + G);
    load_x(gnext, xn);
    __syncthreads();  // (A) A_c complete

    // ---- F: forward products, three components back to back ----
    double g0[3][2], g1[3][2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double* U = SA(c);
      double c0 = 0.0, c1 = 0.0, d0 = 0.0, d1 = 0.0, z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        dmma(c0, c1, U[T::off(w, g, 4 * ks + t)], Dr[ks]);  // x: U_k[j][a] D^T[a][o]
        dmma(d0, d1, Dr[ks], U[T::off(w, 4 * ks + t, g)]);  // y: D[o][b] U_k[b][i]
        dmma(z0, z1, Dr[ks], U[T::off(4 * ks + t, w, g)]);  // z: D[o][c] U_(c, j = w, i)
      }
      g0[c][0] = c0;
      g0[c][1] = c1;
      g1[c][0] = d0;
      g1[c][1] = d1;
      *reinterpret_cast<double2*>(SZ(c) + T::off(g, w, 2 * t)) = make_double2(z0, z1);  // dist Z
    }
    if (!(prm.ablate & 4)) mbar_wait(&qbar, (uint32_t)(it & 1));
    __syncthreads();  // (B) Z_c complete; A_c consumed by the forward products

    // ---- Q: QFunction (qfunction.cpp:135-162), factors once per point pair ----
    {
      const int k = w, sp = T::off(k, g, 2 * t);
      double2 s[6];
      if constexpr (!T::PAD) {
        const int pt = k * 64 + g * 8 + 2 * t;
#pragma unroll
        for (int m = 0; m < 6; ++m) s[m] = *reinterpret_cast<const double2*>(sQD + m * T::P3 + pt);
      } else {
        const int pt = (k * NP + g) * NP + 2 * t;
        const bool v0 = k < NP && g < NP && 2 * t < NP, v1 = k < NP && g < NP && 2 * t + 1 < NP;
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          s[m].x = v0 ? sQD[m * T::NP3 + pt] : 0.0;
          s[m].y = v1 ? sQD[m * T::NP3 + pt + 1] : 0.0;
        }
      }
      double energy = 0.0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double2 z2 = *reinterpret_cast<const double2*>(SZ(c) + sp);
        const double gz[2] = {z2.x, z2.y};
        double v0[2], v1[2], v2[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double a0 = g0[c][h], a1 = g1[c][h], a2 = gz[h];
          const double s00 = h ? s[0].y : s[0].x, s01 = h ? s[1].y : s[1].x;
          const double s02 = h ? s[2].y : s[2].x, s11 = h ? s[3].y : s[3].x;
          const double s12 = h ? s[4].y : s[4].x, s22 = h ? s[5].y : s[5].x;
          v0[h] = s00 * a0 + s01 * a1 + s02 * a2;
          v1[h] = s01 * a0 + s11 * a1 + s12 * a2;
          v2[h] = s02 * a0 + s12 * a1 + s22 * a2;
          energy += a0 * v0[h] + a1 * v1[h] + a2 * v2[h];  // grad u . S grad u
        }
        *reinterpret_cast<double2*>(SA(c) + sp) = make_double2(v0[0], v0[1]);
        *reinterpret_cast<double2*>(SB(c) + sp) = make_double2(v1[0], v1[1]);
        *reinterpret_cast<double2*>(SZ(c) + sp) = make_double2(v2[0], v2[1]);
      }
      dot_acc += prm.coef * energy;
    }
    fence_proxy_async_smem();  // generic reads of the factors before the refill
    __syncthreads();  // (C) V0, V1, V2 complete; factors consumed
    if (tid == 0 && e + G < nsteps && !(prm.ablate & 4)) issue_qdata(e + G);

    // ---- T: transposed products, three components back to back ----
    double y01[3][2], y2z[3][2];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double c0 = 0.0, c1 = 0.0, z0 = 0.0, z1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        dmma(c0, c1, SA(c)[T::off(w, g, 4 * ks + t)], Dc[ks]);  // x^T: V0_k[j][a] D[a][i]
        dmma(c0, c1, Dc[ks], SB(c)[T::off(w, 4 * ks + t, g)]);  // y^T: D^T[j][b] V1_k[b][i]
        dmma(z0, z1, Dc[ks], SZ(c)[T::off(4 * ks + t, w, g)]);  // z^T (dist Z)
      }
      y01[c][0] = c0;
      y01[c][1] = c1;
      y2z[c][0] = z0;
      y2z[c][1] = z1;
    }
    __syncthreads();  // (D) B_c (V1) free
#pragma unroll
    for (int c = 0; c < 3; ++c)
      *reinterpret_cast<double2*>(SB(c) + T::off(g, w, 2 * t)) = make_double2(y2z[c][0], y2z[c][1]);
    __syncthreads();  // (E) z^T in B_c

    // ---- S: combine on dist X, G^T scatter (constrained rows preset by the caller) ----
    if (gcur.active && !(prm.ablate & 2)) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double2 z2 = *reinterpret_cast<const double2*>(SB(c) + T::off(w, g, 2 * t));
        double* yc = prm.y + c * prm.n_L;
        // (padding points have no node: no address is formed for them)
        if (!((gcur.cmask >> 0) & 1u)) red_add(yc + node_of(gcur, 0), prm.coef * (y01[c][0] + z2.x));
        if (!((gcur.cmask >> 1) & 1u)) red_add(yc + node_of(gcur, 1), prm.coef * (y01[c][1] + z2.y));
      }
    }
    // (no trailing barrier: the next element writes A_c (last read in T,
    // before D), Z_c (read in T) and B_c only after its barriers A and B)
    gcur = gnext;
  }

  if (prm.dot_partials) {
    const double s = block_sum<NT>(dot_acc, red_scratch);
    if (tid == 0) prm.dot_partials[blockIdx.x] = s;
    pcg_alpha_epilogue<NT>(prm.fin, red_scratch);
  }
}

}  // namespace hxf
