// K1 (collocated BP5/BP6 fast path): pencil-decomposed fused operator
//   y = G^T D^T S D G x   on GLL-collocated elements (interp1d == I).
//
// Same contract as op_apply_kernel (op_kernel.cuh) — masked gather, RED
// scatter, constrained y = x, fused p.Ap partials — restructured for issue
// efficiency on sm_100a:
//   * every 1-D contraction is a register-resident "pencil": one thread owns a
//     whole x-, y- or z-line of the element and multiplies it by the 1-D
//     derivative matrix held in the kernel-parameter constant bank (DFMA with
//     constant operands, no shared-memory matrix loads);
//   * lines move between threads through two padded shared slabs, updated in
//     place (rows padded to 2 mod 4 doubles, planes skewed by half a bank
//     cycle, so the x-line LDS.128 and the y-line LDS.64 are conflict-free);
//   * the element's geometric factors (6 P^3 doubles) arrive by one bulk
//     async copy (TMA engine, L2 evict_first) issued as soon as the previous
//     element has consumed its factors, i.e. a full transpose phase plus the
//     next gather ahead of use, in a single stage — half the shared memory of
//     a double buffer, so more CTAs (and more bytes in flight) per SM.
// Reference semantics: proj/src/operator.cpp:64-144 (see op_kernel.cuh).
#pragma once
#include "hxf_device.cuh"
#include "hxf_internal.h"

namespace hxf {

__host__ __device__ constexpr int pencil_round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ constexpr int pencil_row_stride(int P) {
  // smallest RS >= P with RS = 2 (mod 4): 16-byte aligned rows whose 8-lane
  // LDS.128 phases fall on distinct bank quads
  return ((P + 1) / 4) * 4 + 2 >= P ? ((P + 1) / 4) * 4 + 2 : ((P + 1) / 4) * 4 + 6;
}

template <int P_, int NC_>
struct PencilTraits {
  static constexpr int P = P_, NC = NC_, PP = P * P, P3 = P * P * P;
  static constexpr int EPB = PP >= 64 ? 1 : (PP == 25 ? 5 : (PP == 36 ? 3 : (PP == 49 ? 2 : 64 / PP)));
  static constexpr int NT = pencil_round_up(EPB * PP, 32);
  static constexpr int RS = pencil_row_stride(P);
  static constexpr int PL = P * RS + 8;  // plane stride: +64 B skews consecutive planes by 16 banks
  static constexpr int SLAB = P * PL;    // doubles per element slab
  static constexpr int QDS = 6 * P3;     // geometric factors per element (even)
  static constexpr int OFF_QD = 0;
  static constexpr int OFF_A = OFF_QD + EPB * QDS;
  static constexpr int OFF_B = OFF_A + EPB * SLAB;
  static constexpr int SMEM_BYTES = (OFF_B + EPB * SLAB) * 8;
};

template <int P>
struct PencilMats {
  double D[P * P];  // grad1d (q = p+1 GLL), row = quadrature point
};

template <class T>
__global__ void __launch_bounds__(T::NT)
    op_pencil_kernel(const OpParams prm, const PencilMats<T::P> mats) {
  constexpr int P = T::P, PP = T::PP, P3 = T::P3, EPB = T::EPB, NT = T::NT, NC = T::NC;
  constexpr int RS = T::RS, PL = T::PL;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t qbar;
  __shared__ double red_scratch[NT / 32 + 1];
  if (prm.stop && *prm.stop) return;

  const int tid = threadIdx.x;
  const int slot = tid / PP;
  const int l = tid - slot * PP;
  const bool active_slot = slot < EPB;
  const int la = l % P, lb = l / P;  // (i,j) | (j,k) | (i,k) depending on the phase
  double* sQD = smem + T::OFF_QD;
  double* SA = smem + T::OFF_A + (active_slot ? slot : 0) * T::SLAB;
  double* SB = smem + T::OFF_B + (active_slot ? slot : 0) * T::SLAB;
  const double* qd_el = sQD + (active_slot ? slot : 0) * T::QDS;

  const int64_t nsteps = (prm.E + EPB - 1) / EPB;
  const int64_t G = gridDim.x;
  uint64_t policy = 0;
  auto issue_qdata = [&](int64_t s) {
    const int64_t e0 = s * EPB;
    const int ne = (int)((prm.E - e0) < EPB ? (prm.E - e0) : EPB);
    const uint32_t bytes = (uint32_t)(ne * T::QDS * 8);
    mbar_arrive_expect_tx(&qbar, bytes);
    bulk_g2s(sQD, prm.qd + e0 * T::QDS, bytes, &qbar, policy);
  };
  if (tid == 0) {
    mbar_init(&qbar, 1);
    fence_mbar_init();
    policy = l2_evict_first_policy();
    if ((int64_t)blockIdx.x < nsteps && !(prm.ablate & 4)) issue_qdata(blockIdx.x);
  }
  __syncthreads();

  const int64_t NXY = prm.NX * prm.NY;
  double dot_acc = 0.0;
  int it = 0;
  for (int64_t step = blockIdx.x; step < nsteps; step += G, ++it) {
    const int64_t e = step * EPB + slot;
    const bool active = active_slot && e < prm.E;
    // node of (i = la, j = lb, k = 0) and whether the element touches the
    // constrained set (structured box boundary, or any bitmask mode)
    int64_t base = 0, ix0 = 0, iy0 = 0, iz0 = 0;
    bool edge = prm.cons_mode != 0;
    if (active && !prm.idx) {
      const int64_t ex = e % prm.nx, r = e / prm.nx, ey = r % prm.ny, ez = r / prm.ny;
      ix0 = ex * (P - 1) + la;
      iy0 = ey * (P - 1) + lb;
      iz0 = ez * (P - 1);
      base = ix0 + prm.NX * iy0 + NXY * iz0;
      if (prm.cons_mode == 1)
        edge = ex == 0 || ey == 0 || ez == 0 || ex == prm.nx - 1 || ey == prm.ny - 1 ||
               (ez + 1) * (P - 1) == prm.NZ - 1;
    }
    auto node_at = [&](int k) -> int64_t {
      return prm.idx ? (int64_t)prm.idx[e * P3 + la + P * (lb + P * k)] : base + k * NXY;
    };
    auto is_cons = [&](int64_t node, int k) -> bool {
      if (!edge) return false;
      if (prm.cons_mode == 2) return (prm.cons_mask[node >> 5] >> (node & 31)) & 1u;
      return ix0 == 0 || ix0 == prm.NX - 1 || iy0 == 0 || iy0 == prm.NY - 1 || iz0 + k == 0 ||
             iz0 + k == prm.NZ - 1;
    };

#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      const double* xc = prm.x + c * prm.n_L;
      double* yc = prm.y + c * prm.n_L;
      if (c > 0 || it > 0) __syncthreads();  // slabs free (previous final phase done)

      // ---- gather z-line (i,j) = (la,lb); masked copy into slab A ----
      double u[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        u[k] = 0.0;
        if (active) {
          const int64_t node = node_at(k);
          u[k] = (prm.ablate & 1) ? 1.0 : (is_cons(node, k) ? 0.0 : __ldg(xc + node));
        }
        if (active_slot) SA[k * PL + lb * RS + la] = u[k];
      }
      __syncthreads();

      // ---- y-pencil (i,k) = (la,lb): g1 = D along y, into slab B ----
      if (active_slot) {
        double col[P];
#pragma unroll
        for (int b = 0; b < P; ++b) col[b] = SA[lb * PL + b * RS + la];
#pragma unroll
        for (int o = 0; o < P; ++o) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < P; ++b) s += mats.D[o * P + b] * col[b];
          SB[lb * PL + o * RS + la] = s;
        }
      }
      __syncthreads();
      // ---- x-pencil (j,k) = (la,lb): g0 = D along x, in place in slab A ----
      if (active_slot) {
        double row[P];
        double* rp = SA + lb * PL + la * RS;
#pragma unroll
        for (int a = 0; a + 1 < P; a += 2) {
          const double2 v = *reinterpret_cast<const double2*>(rp + a);
          row[a] = v.x;
          row[a + 1] = v.y;
        }
        if (P & 1) row[P - 1] = rp[P - 1];
        double g[P];
#pragma unroll
        for (int o = 0; o < P; ++o) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < P; ++a) s += mats.D[o * P + a] * row[a];
          g[o] = s;
        }
#pragma unroll
        for (int a = 0; a + 1 < P; a += 2)
          *reinterpret_cast<double2*>(rp + a) = make_double2(g[a], g[a + 1]);
        if (P & 1) rp[P - 1] = g[P - 1];
      }
      if (c == 0 && !(prm.ablate & 4)) mbar_wait(&qbar, (uint32_t)(it & 1));
      __syncthreads();

      // ---- pointwise: z-derivative from registers + QFunction (qfunction.cpp:135-162) ----
      double v2[P];
#pragma unroll
      for (int k = 0; k < P; ++k) {
        double g2 = 0.0;
#pragma unroll
        for (int cc = 0; cc < P; ++cc) g2 += mats.D[k * P + cc] * u[cc];
        const int sp = k * PL + lb * RS + la;
        const int pt = k * PP + lb * P + la;
        const double g0 = SA[sp], g1 = SB[sp];
        double s00 = 0, s01 = 0, s02 = 0, s11 = 0, s12 = 0, s22 = 0;
        if (active) {
          s00 = qd_el[0 * P3 + pt];
          s01 = qd_el[1 * P3 + pt];
          s02 = qd_el[2 * P3 + pt];
          s11 = qd_el[3 * P3 + pt];
          s12 = qd_el[4 * P3 + pt];
          s22 = qd_el[5 * P3 + pt];
        }
        if (active_slot) {
          SA[sp] = s00 * g0 + s01 * g1 + s02 * g2;
          SB[sp] = s01 * g0 + s11 * g1 + s12 * g2;
        }
        v2[k] = s02 * g0 + s12 * g1 + s22 * g2;
      }
      if (c == NC - 1) fence_proxy_async_smem();  // generic reads of the factors before the refill
      __syncthreads();
      // factors consumed: stream the next step's in while we transpose
      if (c == NC - 1 && tid == 0 && step + G < nsteps && !(prm.ablate & 4)) issue_qdata(step + G);

      // ---- transposed y-pencil (in place, slab B) and x-pencil (in place, slab A) ----
      if (active_slot) {
        double col[P];
#pragma unroll
        for (int b = 0; b < P; ++b) col[b] = SB[lb * PL + b * RS + la];
#pragma unroll
        for (int o = 0; o < P; ++o) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < P; ++b) s += mats.D[b * P + o] * col[b];
          SB[lb * PL + o * RS + la] = s;
        }
        double row[P];
        double* rp = SA + lb * PL + la * RS;
#pragma unroll
        for (int a = 0; a + 1 < P; a += 2) {
          const double2 v = *reinterpret_cast<const double2*>(rp + a);
          row[a] = v.x;
          row[a + 1] = v.y;
        }
        if (P & 1) row[P - 1] = rp[P - 1];
        double t[P];
#pragma unroll
        for (int o = 0; o < P; ++o) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < P; ++a) s += mats.D[a * P + o] * row[a];
          t[o] = s;
        }
#pragma unroll
        for (int a = 0; a + 1 < P; a += 2)
          *reinterpret_cast<double2*>(rp + a) = make_double2(t[a], t[a + 1]);
        if (P & 1) rp[P - 1] = t[P - 1];
      }
      __syncthreads();

      // ---- z^T from registers + combine, G^T scatter ----
      if (active) {
#pragma unroll
        for (int k = 0; k < P; ++k) {
          double s = 0.0;
#pragma unroll
          for (int cc = 0; cc < P; ++cc) s += mats.D[cc * P + k] * v2[cc];
          const int sp = k * PL + lb * RS + la;
          const double yk = prm.coef * (SA[sp] + SB[sp] + s);
          const int64_t node = node_at(k);
          if (prm.ablate & 2) {
            dot_acc += u[k] * yk;
          } else if (is_cons(node, k)) {
            yc[node] = __ldg(xc + node);
          } else {
            red_add(yc + node, yk);
            dot_acc += u[k] * yk;
          }
        }
      }
    }
  }

  if (prm.dot_partials) {
    const double s = block_sum<NT>(dot_acc, red_scratch);
    if (tid == 0) prm.dot_partials[blockIdx.x] = s;
  }
}

}  // namespace hxf
