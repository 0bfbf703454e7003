// K1 (collocated BP5 / BP6, p = 8..15): fused operator on the FP64 tensor
// cores in even-odd form.
//   y = G^T D^T S D G x   on GLL-collocated elements (interp1d == I).
//
// The 1-D derivative matrix of a symmetric node set is centro-antisymmetric,
// D[N-1-o][N-1-a] = -D[o][a] (as is D^T), so every 1-D contraction of a line
// x splits into two half-size products (op_eo.cuh):
//   e[a] = x[a] + x[N-1-a], f[a] = x[a] - x[N-1-a]   (a < N/2; odd N: e[mid] = x[mid])
//   E = Ee e, F = Eo f   (H x H, H = ceil(N/2) <= 8)
//   out[o] = E + F, out[N-1-o] = F - E                (o < H)
// For N = 9..16 the halves fit one 8x8 tile (zero-padded below N = 15), so each
// contraction of 8 lines is 4 DMMA m8n8k4 (two k-steps x {Ee, Eo}) on the FP64
// tensor core instead of ~N^2/2 DFMA lanes each — the line kernel
// (op_line.cuh) it replaces is issue-bound at these orders (BP5 p = 12..15 at
// 0.32-0.41 of HBM, issue-active 23 %).
//
// One element (per component) at a time per CTA of N warps (one per plane
// and row: no warp carries two units across a barrier), one CTA per SM.
// Lane l: g = l>>2, t = l&3 (the mma fragment coordinates).  "dist X" of
// plane k: the lane owns the 8 points (k, R_r, C_q), rows R = {g, N-1-g} and
// columns C = {2t, 2t+1, N-1-2t, N-2-2t} — exactly the rows / columns an
// even-odd product emits for output pair (o, N-1-o), so the x-, y- and
// (through shared memory) z-derivatives of a point meet in one lane.  Warp w
// owns plane w and (for the z-direction, "dist Z") row w.
//   B0  the element's x slab landed (cp.async, issued one item ahead)
//   1   z-derivative of the warp's row (dist Z) -> slab Z
//   2   x- and y-derivatives of the warp's plane in registers, QFunction with
//       the factors staged in shared memory (N <= 14: one bulk copy set per
//       element, issued when the previous element's QFunction consumed its
//       factors, the element after that L2-prefetched) or read from L2
//       (N = 15, 16: bulk-prefetched one element ahead); V0 -> slab U (in
//       place), V1 -> slab B, V2 -> slab Z
//   3   x^T + y^T of the plane -> slab U (in place); then the next item's
//       gather into slab B, z^T of the row in registers and the scatter:
//       y = U + z^T in dist Z, FP64 RED
// Slabs are [k][j][16] (rows padded to 16 doubles) with the column XOR-
// swizzled by 4 * (perm(j & 3) ^ perm(k & 3)), perm swapping the two bits:
// every fragment load (8 rows x 4 columns, 4 rows x 8 columns, 4 planes x 8
// columns) and every dist X / dist Z pair access is at its wavefront minimum.
// Reference semantics: proj/src/operator.cpp:64-144 (see op_kernel.cuh).
#pragma once
#include "hxf_device.cuh"
#include "hxf_internal.h"
#include "op_dmma.cuh"  // dmma()
#include "pcg_device.cuh"

#ifndef HXF_EO_MINB  // CTAs per SM the register budget targets (0: two for N <= 11)
#define HXF_EO_MINB 1
#endif
namespace hxf {

template <int N_, int NC_>
struct EoTraits {
  static constexpr int N = N_, NC = NC_, NN = N_ * N_, N3 = N_ * N_ * N_;
  static constexpr int H = (N_ + 1) / 2, HI = N_ / 2;
  static constexpr bool ODD = (N_ & 1) != 0;
  static_assert(N_ >= 9 && N_ <= 16, "even-odd halves of 5..8 fit one 8x8 DMMA tile");
  // one warp per plane (x / y products, QFunction, x^T / y^T) and per row
  // (z and z^T products): no warp holds two units across a barrier
  static constexpr int NW = N_, NT = 32 * N_;
  static constexpr int SLAB = N_ * N_ * 16;  // doubles (rows padded to 16)
  static constexpr int QDS = 6 * N3;         // geometric factors per element
  // QS: the element's factors staged in shared memory by bulk copies (TMA
  // engine), issued as soon as the previous element's QFunction consumed
  // them; N = 15, 16 do not fit (162 / 196 KB) and read them from L2 instead
  // (measured and dropped for N = 16: staging the first 8 rows of every factor
  // plane with 96 bulk copies per element, BP5 p = 15 198 -> 235 us)
  static constexpr int SLABS_BYTES = 3 * SLAB * 8;
  static constexpr bool QS = SLABS_BYTES + QDS * 8 + 4096 <= 227 * 1024;
  static constexpr int SMEM_BYTES = SLABS_BYTES + (QS ? QDS * 8 : 0);
  // one CTA per SM (~128-166 registers per thread).  Measured with two (N <=
  // 11, 96 / 80 registers, small spills; HXF_EO_MINB=0 at build time): BP5
  // p = 8 / 9 652 -> 512 / 543 -> 447 us but p = 10 388 -> 425 us — still far
  // behind the line kernel (205 / 257 / 264 us) there, so not dispatched
  static constexpr int MINB = HXF_EO_MINB > 0 ? HXF_EO_MINB
                              : ((N_ <= 11 && 2 * (SMEM_BYTES + 3072) <= 228 * 1024) ? 2 : 1);
  __device__ static __forceinline__ int perm(int x) { return ((x & 1) << 1) | ((x >> 1) & 1); }
  __device__ static __forceinline__ int off(int k, int j, int i) {
    return (k * N_ + j) * 16 + (i ^ (4 * (perm(j & 3) ^ perm(k & 3))));
  }
};

__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p));
  return v;
}

template <class T>
__global__ void __launch_bounds__(T::NT, T::MINB) op_dmmaeo_kernel(const __grid_constant__ OpParams prm) {
  constexpr int N = T::N, NN = T::NN, N3 = T::N3, H = T::H, HI = T::HI, NC = T::NC, NT = T::NT;
  extern __shared__ __align__(128) double eo_smem[];
  __shared__ double red_scratch[NT / 32 + 1];
  pdl_wait();  // x, y, stop and the PCG state come from the previous kernels
  if (prm.stop && *prm.stop) return;

  const bool skipc = (prm.ablate & 16) != 0;  // measurement-only: no tensor-core products
  const int tid = threadIdx.x;
  const int w = tid >> 5, l = tid & 31, g = l >> 2, t = l & 3;
  double* SU = eo_smem;            // U, then V0, then x^T + y^T
  double* SB = eo_smem + T::SLAB;  // V1; the next item's U
  double* SZ = eo_smem + 2 * T::SLAB;

  // even-odd fragments of D and D^T: lane holds E[g][4ks+t] (A operand of a
  // row product, B operand of a column product — the same values)
  // (kept in a 2 KB shared table, read at the start of the phase that uses
  // them: 8 fewer live registers across the other phases)
  __shared__ double2 efrag[4][32];  // {Ee, Eo} of D: [0] k-step 0, [1] k-step 1; of D^T: [2], [3]
  if (tid < 32) {
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const int a = 4 * ks + t, o = g;
      auto Dm = [&](int r, int c) { return __ldg(prm.D + r * N + c); };
      const bool ein = o < H && a < H, oin = o < H && a < HI;
      efrag[ks][l] = make_double2(ein ? (a < HI ? 0.5 * (Dm(o, a) + Dm(o, N - 1 - a)) : Dm(o, HI)) : 0.0,
                                  oin ? 0.5 * (Dm(o, a) - Dm(o, N - 1 - a)) : 0.0);
      efrag[2 + ks][l] = make_double2(ein ? (a < HI ? 0.5 * (Dm(a, o) + Dm(N - 1 - a, o)) : Dm(HI, o)) : 0.0,
                                      oin ? 0.5 * (Dm(a, o) - Dm(N - 1 - a, o)) : 0.0);
    }
  }
  auto frags = [&](int which, double* me, double* mo) {  // which 0: D, 1: D^T
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      const double2 v = efrag[2 * which + ks][l];
      me[ks] = v.x;
      mo[ks] = v.y;
    }
  };
  const int R0 = g, R1 = N - 1 - g;
  const bool rv0 = g < H, rv1 = g < HI;
  const int C0 = 2 * t, C1 = 2 * t + 1, C2 = N - 1 - 2 * t, C3 = N - 2 - 2 * t;
  const bool cv[4] = {2 * t < H, 2 * t + 1 < H, 2 * t < HI, 2 * t + 1 < HI};
  const int Cq[4] = {C0, C1, C2, C3};

  // even-odd operand pair of a line (x0 = x[a], x1 = x[N-1-a], a = 4ks+t)
  auto evod = [&](double x0, double x1, int a, double& e, double& f) {
    e = a < HI ? x0 + x1 : ((T::ODD && a == HI) ? x0 : 0.0);
    f = a < HI ? x0 - x1 : 0.0;
  };
  // column product of plane k: out[j][o] = sum_a S[k][j][a] M[o][a], rows R0 / R1
  auto colop = [&](const double* S, int k, const double* me, const double* mo, double* out) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int row = mt ? R1 : R0;
      double pe0 = 0.0, pe1 = 0.0, po0 = 0.0, po1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int a = 4 * ks + t;
        double e, f;
        evod(S[T::off(k, row, a)], S[T::off(k, row, N - 1 - a)], a, e, f);
        if (!skipc) dmma(pe0, pe1, e, me[ks]);
        if (!skipc) dmma(po0, po1, f, mo[ks]);
      }
      out[mt * 4 + 0] = pe0 + po0;
      out[mt * 4 + 1] = pe1 + po1;
      out[mt * 4 + 2] = po0 - pe0;
      out[mt * 4 + 3] = po1 - pe1;
    }
  };
  // row product: out[o][c] = sum_b M[o][b] X(b, c); slots (r, q) = (row R_r, column C_q)
  auto rowop = [&](auto X, const double* me, const double* mo, double* out) {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int cb = nt ? N - 1 - g : g;  // this lane's B-fragment column
      double pe0 = 0.0, pe1 = 0.0, po0 = 0.0, po1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        const int b = 4 * ks + t;
        double e, f;
        evod(X(b, cb), X(N - 1 - b, cb), b, e, f);
        if (!skipc) dmma(pe0, pe1, me[ks], e);
        if (!skipc) dmma(po0, po1, mo[ks], f);
      }
      out[nt * 2 + 0] = pe0 + po0;
      out[nt * 2 + 1] = pe1 + po1;
      out[4 + nt * 2 + 0] = po0 - pe0;
      out[4 + nt * 2 + 1] = po1 - pe1;
    }
  };
  auto valid = [&](int s) { return (s < 4 ? rv0 : rv1) && cv[s & 3]; };
  // the lane's two column pairs of a row, in memory order: pair 0 = (C0, C1)
  // (16-byte aligned), pair 1 = (C3, C2) (aligned for even N); slots lo / hi
  auto ld_pair = [&](const double* S, int k, int R, int hp, double& lo, double& hi) {
    if (hp == 0 || !T::ODD) {
      const double2 v = *reinterpret_cast<const double2*>(S + T::off(k, R, hp ? C3 : C0));
      lo = v.x;
      hi = v.y;
    } else {
      lo = S[T::off(k, R, C3)];
      hi = S[T::off(k, R, C2)];
    }
  };
  // reads only the valid slots (0 otherwise): in a phase that rewrites the
  // points in place, an invalid slot aliases a point another lane rewrites
  auto ld_pair_v = [&](const double* S, int k, int R, int hp, double& lo, double& hi, bool vlo,
                       bool vhi) {
    if ((hp == 0 || !T::ODD) && vlo && vhi) {
      const double2 v = *reinterpret_cast<const double2*>(S + T::off(k, R, hp ? C3 : C0));
      lo = v.x;
      hi = v.y;
    } else {
      lo = vlo ? S[T::off(k, R, hp ? C3 : C0)] : 0.0;
      hi = vhi ? S[T::off(k, R, hp ? C2 : C1)] : 0.0;
    }
  };
  // stores only the valid slots (an invalid slot aliases a point another
  // slot owns)
  auto st_pair = [&](double* S, int k, int R, int hp, double lo, double hi, bool vlo, bool vhi) {
    if ((hp == 0 || !T::ODD) && vlo && vhi) {
      *reinterpret_cast<double2*>(S + T::off(k, R, hp ? C3 : C0)) = make_double2(lo, hi);
    } else {
      if (vlo) S[T::off(k, R, hp ? C3 : C0)] = lo;
      if (vhi) S[T::off(k, R, hp ? C2 : C1)] = hi;
    }
  };
  // slot numbers of pair hp: lo, hi
  auto slo = [](int hp) { return hp ? 3 : 0; };
  auto shi = [](int hp) { return hp ? 2 : 1; };
  // store 8 slots of row-pair (R0, R1) at plane k (dist X) or of row j with
  // planes (R0, R1) (dist Z)
  auto st_slots_x = [&](double* S, int k, const double* v) {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int hp = 0; hp < 2; ++hp)
        st_pair(S, k, r ? R1 : R0, hp, v[4 * r + slo(hp)], v[4 * r + shi(hp)], valid(4 * r + slo(hp)),
                valid(4 * r + shi(hp)));
  };
  auto st_slots_z = [&](double* S, int j, const double* v) {
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int hp = 0; hp < 2; ++hp) {
        const int R = r ? R1 : R0;
        const int sl = 4 * r + slo(hp), sh = 4 * r + shi(hp);
        if ((hp == 0 || !T::ODD) && valid(sl) && valid(sh)) {
          *reinterpret_cast<double2*>(S + T::off(R, j, hp ? C3 : C0)) = make_double2(v[sl], v[sh]);
        } else {
          if (valid(sl)) S[T::off(R, j, hp ? C3 : C0)] = v[sl];
          if (valid(sh)) S[T::off(R, j, hp ? C2 : C1)] = v[sh];
        }
      }
  };

  const int64_t nsteps = prm.E;
  const int64_t G = gridDim.x;
  const int64_t NXY = prm.NX * prm.NY;
  auto elem = [&](int64_t s) {
    const int64_t k = prm.rev ? nsteps - 1 - s : s;
    return prm.elist ? (int64_t)__ldg(prm.elist + k) : k;
  };
  struct Geo {
    int64_t e, base;
    int ix0, iy0, iz0;
    bool bnd;  // touches a constrained box face
  };
  const FastDiv divx((uint32_t)prm.nx), divy((uint32_t)prm.ny);
  auto geometry = [&](int64_t s) {
    Geo q{};
    q.e = elem(s);
    const uint32_t e32 = (uint32_t)q.e, r = divx.div(e32), ez = divy.div(r);
    const uint32_t ex = e32 - r * (uint32_t)prm.nx, ey = r - ez * (uint32_t)prm.ny;
    q.ix0 = (int)(ex * (N - 1));
    q.iy0 = (int)(ey * (N - 1));
    q.iz0 = (int)(ez * (N - 1));
    q.base = q.ix0 + prm.NX * q.iy0 + NXY * q.iz0;
    const int f = prm.cons_mode == 1 ? prm.bnd_faces : 0;
    q.bnd = ((f & 1) && q.ix0 == 0) || ((f & 2) && q.ix0 + N - 1 == prm.NX - 1) ||
            ((f & 4) && q.iy0 == 0) || ((f & 8) && q.iy0 + N - 1 == prm.NY - 1) ||
            ((f & 16) && q.iz0 == 0) || ((f & 32) && q.iz0 + N - 1 == prm.NZ - 1);
    return q;
  };
  // The element's x slab by rows: thread 2r + h copies half h (columns
  // 8h .. min(N, 8h + 8)) of row r = (k, j) with cp.async, in 16-byte pairs
  // when the global row is 16-byte aligned (the slab keeps (2m, 2m+1) pairs
  // adjacent: the swizzle moves 4-double groups); and it masks those same
  // points after its own copies landed.
  // (measured: per-point copies with the index math per point cost ~12 % of
  // the kernel's instructions at N = 14)
  const bool gthr = tid < 2 * NN;
  const int grow = tid >> 1, gk = grow / N, gj = grow - gk * N;
  const int gc0 = (tid & 1) * 8, gc1 = gc0 + 8 < N ? gc0 + 8 : N;
  const int ghx = 4 * (T::perm(gj & 3) ^ T::perm(gk & 3));
  auto issue_gather = [&](const Geo& q, int c, double* dst) {
    if ((prm.ablate & 1) || !gthr) return;
    const double* g = prm.x + c * prm.n_L + q.base + prm.NX * gj + NXY * gk;
    double* drow = dst + (gk * N + gj) * 16;
    if ((reinterpret_cast<uintptr_t>(g) & 15u) == 0) {
      int col = gc0;
      for (; col + 1 < gc1; col += 2) cp_async16(drow + (col ^ ghx), g + col);
      if (col < gc1) cp_async8(drow + (col ^ ghx), g + col);
    } else {
      for (int col = gc0; col < gc1; ++col) cp_async8(drow + (col ^ ghx), g + col);
    }
  };
  // own points of the gather: zero the constrained ones (y = x stored first
  // for a single apply that zero-filled y)
  auto mask_gather = [&](const Geo& q, int c, double* dst) {
    if (!q.bnd || !gthr) return;
    const int f = prm.bnd_faces;
    const int64_t iy = q.iy0 + gj, iz = q.iz0 + gk;
    const bool row_all = ((f & 4) && iy == 0) || ((f & 8) && iy == prm.NY - 1) ||
                         ((f & 16) && iz == 0) || ((f & 32) && iz == prm.NZ - 1);
    const bool lo = (f & 1) && q.ix0 == 0, hi = (f & 2) && q.ix0 + N - 1 == prm.NX - 1;
    double* drow = dst + (gk * N + gj) * 16;
    for (int col = gc0; col < gc1; ++col) {
      if (!(row_all || (col == 0 && lo) || (col == N - 1 && hi))) continue;
      double* p = drow + (col ^ ghx);
      if (prm.cons_store) prm.y[c * prm.n_L + q.base + col + prm.NX * gj + NXY * gk] = *p;
      *p = 0.0;
    }
  };

  __shared__ __align__(8) uint64_t qbar;
  double* SQ = eo_smem + 3 * T::SLAB;  // staged factors (T::QS)
  auto issue_qdata = [&](int64_t e) {  // bulk copies of <= 32 KB (16-byte multiples)
    constexpr uint32_t total = T::QDS * 8, chunk = 32768;
    mbar_arrive_expect_tx(&qbar, total);
    const uint64_t pol = l2_evict_first_policy();
    const char* src = reinterpret_cast<const char*>(prm.qd + e * T::QDS);
    char* dst = reinterpret_cast<char*>(SQ);
#pragma unroll 1
    for (uint32_t o = 0; o < total; o += chunk)
      bulk_g2s(dst + o, src + o, total - o < chunk ? total - o : chunk, &qbar, pol);
  };
  const int k = w, j = w;  // this warp's plane and row
  double dot_acc = 0.0;
  int64_t s = blockIdx.x;
  Geo cur{};
  if constexpr (T::QS) {
    if (tid == 0) {
      mbar_init(&qbar, 1);
      fence_mbar_init();
    }
    __syncthreads();  // mbarrier initialised before any thread uses it
  }
  if (s < nsteps) {
    cur = geometry(s);
    if (tid == 0 && !(prm.ablate & 4)) {
      if constexpr (T::QS) {
        issue_qdata(cur.e);
        if (s + G < nsteps) bulk_prefetch_l2(prm.qd + elem(s + G) * T::QDS, (uint32_t)(T::QDS * 8));
      } else {
        bulk_prefetch_l2(prm.qd + cur.e * T::QDS, (uint32_t)(T::QDS * 8));
      }
    }
    issue_gather(cur, 0, SU);
  }
  int it = 0;
#pragma unroll 1
  for (; s < nsteps; s += G, ++it) {
    const bool has_next = s + G < nsteps;
    // factors ahead: HBM -> L2 (staged: the element after next, whose bulk
    // copy is issued during the next element)
    if (tid == 0 && !(prm.ablate & 4)) {
      const int64_t pf = s + (T::QS ? 2 : 1) * G;
      if (pf < nsteps) bulk_prefetch_l2(prm.qd + elem(pf) * T::QDS, (uint32_t)(T::QDS * 8));
    }
    Geo nxt = cur;
    const double* qe = T::QS ? SQ : prm.qd + cur.e * T::QDS;
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      double* yc = prm.y + c * prm.n_L;
      cp_async_wait_all();
      mask_gather(cur, c, SU);
      __syncthreads();  // B0: U complete

      double fe[2], fo[2];
      frags(0, fe, fo);
      // ---- 1: z-derivative of this warp's row (dist Z) -> slab Z ----
      {
        double out[8];
        rowop([&](int b, int col) { return SU[T::off(b, j, col)]; }, fe, fo, out);
        st_slots_z(SZ, j, out);
      }
      __syncthreads();  // B1: G2 complete

      // ---- 2: x / y derivatives of this warp's plane, QFunction (qfunction.cpp:135-162) ----
      double energy = 0.0;
      {
        // factors of step st = (row r = st >> 1, column pair hp = st & 1)
        auto load_sv = [&](int st, double (*sv)[2]) {
          const int R = (st >> 1) ? R1 : R0, hp = st & 1;
          const double* qp = qe + k * NN + R * N;
#pragma unroll
          for (int m = 0; m < 6; ++m) {
            if (prm.ablate & 4) {  // measurement-only: no factor traffic
              sv[m][0] = sv[m][1] = 1.0 + m;
            } else if constexpr (T::QS && !T::ODD) {
              const double2 a = *reinterpret_cast<const double2*>(qp + m * N3 + (hp ? C3 : C0));
              sv[m][0] = a.x;
              sv[m][1] = a.y;
            } else if constexpr (T::QS) {
              sv[m][0] = qp[m * N3 + (hp ? C3 : C0)];
              sv[m][1] = qp[m * N3 + (hp ? C2 : C1)];
            } else if constexpr (!T::ODD) {  // (odd N: factor rows not 16-byte aligned)
              const double2 a = __ldg(reinterpret_cast<const double2*>(qp + m * N3 + (hp ? C3 : C0)));
              sv[m][0] = a.x;
              sv[m][1] = a.y;
            } else {
              sv[m][0] = __ldg(qp + m * N3 + (hp ? C3 : C0));
              sv[m][1] = __ldg(qp + m * N3 + (hp ? C2 : C1));
            }
          }
        };
        // (global factors: software-pipelined one step ahead, step 0 under the
        // DMMA work; staged factors: loaded at their step, fewer live registers)
        double sva[6][2], svb[6][2];
        if constexpr (T::QS) {
          if (c == 0 && !(prm.ablate & 4)) mbar_wait(&qbar, (uint32_t)(it & 1));
        } else {
          load_sv(0, sva);
        }
        double g0[8], g1[8];
        colop(SU, k, fe, fo, g0);
        rowop([&](int b, int col) { return SU[T::off(k, b, col)]; }, fe, fo, g1);
        __syncwarp();  // every lane's reads of plane k before V0 replaces it
#pragma unroll
        for (int st = 0; st < 4; ++st) {
          const int r = st >> 1, hp = st & 1;
          const int R = r ? R1 : R0;
          double (*sv)[2] = (st & 1) ? svb : sva;
          if constexpr (T::QS) {
            load_sv(st, sv);
          } else {
            if (st < 3) load_sv(st + 1, (st & 1) ? sva : svb);
          }
          const int lo = slo(hp), hi = shi(hp);
          double z[2], v0[2], v1[2], v2[2];
          ld_pair_v(SZ, k, R, hp, z[0], z[1], valid(r * 4 + lo), valid(r * 4 + hi));
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int sl = r * 4 + (h ? hi : lo);
            const double a0 = g0[sl], a1 = g1[sl], a2 = z[h];
            const double s00 = sv[0][h], s01 = sv[1][h], s02 = sv[2][h];
            const double s11 = sv[3][h], s12 = sv[4][h], s22 = sv[5][h];
            v0[h] = s00 * a0 + s01 * a1 + s02 * a2;
            v1[h] = s01 * a0 + s11 * a1 + s12 * a2;
            v2[h] = s02 * a0 + s12 * a1 + s22 * a2;
            // p.(A p) over free nodes = sum_points grad u . S grad u
            if (valid(sl)) energy += a0 * v0[h] + a1 * v1[h] + a2 * v2[h];
          }
          const bool vl = valid(r * 4 + lo), vh = valid(r * 4 + hi);
          st_pair(SU, k, R, hp, v0[0], v0[1], vl, vh);
          st_pair(SB, k, R, hp, v1[0], v1[1], vl, vh);
          st_pair(SZ, k, R, hp, v2[0], v2[1], vl, vh);
        }
      }
      dot_acc += prm.coef * energy;
      if (T::QS && c == NC - 1) fence_proxy_async_smem();  // factor reads before the refill
      __syncthreads();  // B2: V0, V1, V2 complete; staged factors consumed
      if (T::QS && c == NC - 1 && tid == 0 && has_next && !(prm.ablate & 4))
        issue_qdata(elem(s + G));

      double te[2], to[2];
      frags(1, te, to);
      // ---- 3: x^T + y^T of this warp's plane -> slab U (in place) ----
      {
        double ya[8], yb[8];
        colop(SU, k, te, to, ya);
        rowop([&](int b, int col) { return SB[T::off(k, b, col)]; }, te, to, yb);
#pragma unroll
        for (int q = 0; q < 8; ++q) ya[q] += yb[q];
        __syncwarp();  // every lane's reads of plane k of U before the sums replace it
        st_slots_x(SU, k, ya);
      }
      __syncthreads();  // B3: x^T + y^T complete; slab B consumed

      // next item's slab into B (lands while this one scatters / the next computes)
      if (c + 1 < NC) {
        issue_gather(cur, c + 1, SB);
      } else if (has_next) {
        nxt = geometry(s + G);
        issue_gather(nxt, 0, SB);
      }
      // ---- z^T of this warp's row (slab Z holds V2 until the next item's
      //      phase 1) and the scatter in dist Z: y = coef (x^T + y^T + z^T),
      //      FP64 RED ----
      {
        const int f = prm.bnd_faces;
        double y2[8];
        rowop([&](int b, int col) { return SZ[T::off(b, j, col)]; }, te, to, y2);
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int R = r ? R1 : R0;
          double u[4];
          ld_pair(SU, R, j, 0, u[0], u[1]);  // (dist Z: plane R, row j)
          ld_pair(SU, R, j, 1, u[3], u[2]);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (!valid(4 * r + q)) continue;
            const int C = Cq[q];
            const double yv = prm.coef * (u[q] + y2[4 * r + q]);
            bool cons = false;
            if (cur.bnd) {
              const int64_t ix = cur.ix0 + C, iy = cur.iy0 + j, iz = cur.iz0 + R;
              cons = ((f & 1) && ix == 0) || ((f & 2) && ix == prm.NX - 1) ||
                     ((f & 4) && iy == 0) || ((f & 8) && iy == prm.NY - 1) ||
                     ((f & 16) && iz == 0) || ((f & 32) && iz == prm.NZ - 1);
            }
            // constrained rows (y = x) are preset by the caller
            if (!cons && !(prm.ablate & 2)) red_add(yc + cur.base + C + prm.NX * j + NXY * R, yv);
          }
        }
      }
      double* tmp = SU;
      SU = SB;
      SB = tmp;
    }
    cur = nxt;
  }
  if (prm.dot_partials) {
    const double sum = block_sum<NT>(dot_acc, red_scratch);
    if (tid == 0) prm.dot_partials[blockIdx.x] = sum;
    pcg_alpha_epilogue<NT>(prm.fin, red_scratch);
  }
}

}  // namespace hxf
