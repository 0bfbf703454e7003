// K1 (line kernel): fused operator  y = G^T B^T D B G x  for the interpolating
// bases (BP1-BP4, q = p+2 Gauss points), one-component collocated p != 7 (BP5)
// and three-component p >= 10 / p = 3 (BP6).
//
// Every 1-D contraction is a register "line": one thread loads the Q (or P)
// values of one line of the element's slab and applies the 1-D matrix in
// even-odd form (op_eo.cuh: half-size tables broadcast from shared memory as
// LDS.128 rows, half the multiply-adds of the plain product; on sm_100 DFMA
// cannot take an FP64 constant-bank operand, so kernel-parameter matrices
// would cost a uniform-register move per use) and writes the line back.
// Phases (one __syncthreads between each):
//   1  x-interp  thread (j,k) gathers its node x-line straight from global
//      memory (software-pipelined one element ahead) -> S0 [k][j][qi]
//   2  y-interp  thread (qi,k)                        -> S1 [k][qj][qi]
//   3  z-interp  thread (qi,qj): u_q column in registers, -> S2, and (q <= 10)
//      the z-derivative of it in registers
//   4  x / y derivatives of S2 (thread (a,b) owns one x-line and one y-line)
//   5  QFunction per column, geometric factors loaded directly from global
//      memory (L2-prefetched one element ahead with cp.async.bulk.prefetch),
//      v0 / v1 in place, v2 in registers (q > 10: z-derivative recomputed here
//      from the S2 column, v2 back into S2); p.(A p) as grad u . S grad u
//   6  x^T / y^T derivatives in place
//   7  column: sum of the three, z^T interp               -> S2 [c][qj][qi]
//   8  y^T interp thread (qi,c)                         -> S1 [c][j][qi]
//   9  x^T interp thread (j,c), FP64 RED scatter of its node x-line
// Mass (BP1/2) skips 4 and 6 and fuses 3-5-7 in registers; collocated skips
// the interpolation phases (the column thread gathers / scatters its z-line).
// Compared with op_apply_kernel (op_kernel.cuh), the slabs need 3 Q^3 doubles
// and no staged geometric factors, so 4-6 CTAs fit per SM instead of 1-2.
// Reference semantics: proj/src/operator.cpp:64-144, contraction.cpp:248-332,
// qfunction.cpp:124-162.
#pragma once
// z-derivative kept in registers up to q = 10 (measured: q = 12 in registers spills,
// BP5 p=11 K1 363 -> 261 us and BP3 p=15 574 -> 505 us with the late form)
// threads per CTA targeted for q <= 4 (several elements per CTA; measured 64 ahead
// of 128 by 2-8 % for q = 2..4 and of 256 by 5-15 %), 128 for q = 5..7
// staged geometric factors up to this many KB per CTA step (0: always global;
// measured 72: BP5 p=10 -9 % but BP5 p=9 / BP3 p=8 +5..6 %)
// (three components: 112 measured mixed for BP6 p = 10-15, -12..+18 %)
#ifndef HXF_LINE_QSMEM_MAXKB3
#define HXF_LINE_QSMEM_MAXKB3 40
#endif
#ifndef HXF_LINE_QSMEM_MAXKB
#define HXF_LINE_QSMEM_MAXKB 40
#endif
#ifndef HXF_LINE_SMALL_NT
#define HXF_LINE_SMALL_NT 64
#endif
// late-form QFunction unroll (measured 4: -7..+11 % across q = 11-16, kept 2)
#ifndef HXF_LINE_QF_UNROLL
#define HXF_LINE_QF_UNROLL 2
#endif
#ifndef HXF_LINE_EARLY_Q
#define HXF_LINE_EARLY_Q 10
#endif
#ifndef HXF_LINE_REGS
#define HXF_LINE_REGS 128
#endif
#include "hxf_device.cuh"
#include "hxf_internal.h"
#include "op_eo.cuh"
#include "op_kernel.cuh"
#include "pcg_device.cuh"

namespace hxf {

template <int P_, int Q_, int NC_, int QK_, bool INTERP_>
struct LineTraits {
  static constexpr int P = P_, Q = Q_, NC = NC_, QK = QK_;
  // z-derivative / v2 of the column kept in registers across phases 4-7
  // (measured faster at q = 9); larger q recompute it from S2 in phase 5
  static constexpr bool EARLY = Q <= HXF_LINE_EARLY_Q;
  static constexpr int QFU = HXF_LINE_QF_UNROLL;  // late-form QFunction unroll
  static constexpr bool INTERP = INTERP_;
  static constexpr bool DIFF = QK == 1;  // one qdata kind per launch (1 diffusion, 2 mass)
  static constexpr int QQ = Q * Q, Q3 = Q * Q * Q, P3 = P * P * P;
  // elements per CTA at q = 9 as a build knob (measured: 2 loses 4-10 % on BP1/3/5,
  // wins 8 % on BP4 only)
#ifndef HXF_LINE_EPB81
#define HXF_LINE_EPB81 1
#endif
  static constexpr int EPB =
      QQ == 81 ? HXF_LINE_EPB81 : (QQ >= 64 ? 1 : ((QQ <= 16 ? HXF_LINE_SMALL_NT : 128) / QQ));
  static constexpr int NT = round_up(EPB * QQ, 32);
  // register target per thread (measured: 112 / 96 targets lose up to 27 % at
  // q = 9 and 10 to spills; 128 gives 5 CTAs of 3 warps at q = 9)
  static constexpr int REGT = HXF_LINE_REGS;
  static constexpr int MINB = (65536 / (NT * REGT)) < 1 ? 1 : (65536 / (NT * REGT) > 8 ? 8 : 65536 / (NT * REGT));
  // odd row stride: x-line (stride RS across lanes) and column / y-line
  // (consecutive across lanes) accesses are all conflict-free (measured: a
  // 16-byte aligned RS = 2 mod 4 with LDS.128 x-lines is 20 % slower at q = 9)
  static constexpr int RS = Q | 1;
  static constexpr int SLAB = Q * Q * RS;
  static constexpr int NQD = DIFF ? 6 : 1;
  static constexpr int QDS = round_up(NQD * Q3, 2);  // padded doubles per element
  // 1-D matrices in shared memory, 16-byte rows (broadcast LDS.128 row loads):
  // D [Q][RQ] (late z-derivative form) and the even-odd tables below
  static constexpr int RQ = round_up(Q, 2);
  static constexpr int OFF_D = 0;
  // even-odd tables (centro-symmetric bases: M[NO-1-o][NI-1-a] = +-M[o][a]):
  // row o < ceil(NO/2) = [ (M[o][a] + M[o][a'])/2 (a < NI/2) | M[o][NI/2] (odd NI)
  // | (M[o][a] - M[o][a'])/2 ], a' = NI-1-a, for B, B^T, D, D^T
  static constexpr int OFF_EBF = round_up(OFF_D + Q * RQ, 2);           // B   (Q x P)
  static constexpr int OFF_EBT = OFF_EBF + ((Q + 1) / 2) * eo_row_stride(P);    // B^T (P x Q)
  static constexpr int OFF_EDF = OFF_EBT + ((P + 1) / 2) * eo_row_stride(Q);    // D   (Q x Q)
  static constexpr int OFF_EDT = OFF_EDF + ((Q + 1) / 2) * eo_row_stride(Q);    // D^T (Q x Q)
  static constexpr int OFF_S = round_up(OFF_EDT + ((Q + 1) / 2) * eo_row_stride(Q), 2);
  // diffusion, one component, factors of a step small enough: stage them in
  // shared memory with one bulk async copy per step (TMA engine), refilled
  // right after the QFunction consumed them, instead of per-point global loads
  // (measured, K1 at 1e7 DOFs: BP5 p = 4, 5, 6, 8 -13..14 %, BP3 p = 3, 4, 5, 7
  // -2..5 %; q <= 4 and BP3 p = 6 lose 2..8 % and keep the global loads)
  // (mass: interpolating bases only, where a barrier follows the QFunction)
  // (collocated q = 11 stages its 64 KB too: measured BP5 p = 10 264 -> 239 us,
  // BP6 p = 10 289 -> 270 us; with a 112 KB limit everywhere BP5 p = 9 / 11 and
  // BP3 p = 8, 10, 11 lose 5..34 %)
  static constexpr bool QS = (DIFF || INTERP_) && Q >= 5 && !(INTERP_ && Q == 8) &&
                             (EPB * QDS * 8 <= (NC == 3 ? HXF_LINE_QSMEM_MAXKB3 : HXF_LINE_QSMEM_MAXKB) * 1024 ||
                              (DIFF && !INTERP_ && Q == 11));
  static constexpr int OFF_QS = round_up(OFF_S + EPB * 3 * SLAB, 2);
  static constexpr int SMEM_BYTES = (OFF_QS + (QS ? EPB * QDS : 0)) * 8;
  __device__ static __forceinline__ int off(int k, int j, int i) { return (k * Q + j) * RS + i; }
};

// Placement of one gather/scatter line of an element: node(n) = base + n*step
// (structured box) or idx[tab + n*tstep] (int32 table); bit n of cmask: node
// n of the line is constrained.
struct LineGeo {
  int64_t base, step;
  int64_t tab;
  int tstep;
  uint32_t cmask;
  bool active;
};

// a contiguous slab line (x-line) to / from registers
template <int N>
__device__ __forceinline__ void ld_line(const double* src, double* d) {
#pragma unroll
  for (int a = 0; a < N; ++a) d[a] = src[a];
}
template <int N>
__device__ __forceinline__ void st_line(double* dst, const double* d) {
#pragma unroll
  for (int a = 0; a < N; ++a) dst[a] = d[a];
}

// Phases 4 / 6: the x-line (b, a, :) of sx and the y-line (b, :, a) of sy
// through the same Q x Q matrix M (rows m + o*RQ), one broadcast row load
// feeding both lines; results to the same lines of dx / dy (in place safe:
// both lines are read before the first write).
template <class T>
__device__ __forceinline__ void line_pair(const double* tab, const double* sx, const double* sy,
                                          double* dx, double* dy, int a, int b) {
  // tab: even-odd table of a Q x Q derivative matrix (S = -1)
  constexpr int Q = T::Q, HI = Q / 2, HO = (Q + 1) / 2, L = 2 * HI + 1, RT = (L + 1) / 2 * 2;
  double ex[HI], fx[HI], ey[HI], fy[HI], mx = 0.0, my = 0.0;
#pragma unroll
  for (int i = 0; i < HI; ++i) {
    const double x0 = sx[T::off(b, a, i)], x1 = sx[T::off(b, a, Q - 1 - i)];
    const double y0 = sy[T::off(b, i, a)], y1 = sy[T::off(b, Q - 1 - i, a)];
    ex[i] = x0 + x1;
    fx[i] = x0 - x1;
    ey[i] = y0 + y1;
    fy[i] = y0 - y1;
  }
  if constexpr (Q & 1) {
    mx = sx[T::off(b, a, HI)];
    my = sy[T::off(b, HI, a)];
  }
#pragma unroll
  for (int o = 0; o < HO; ++o) {
    double row[L];
    line_row<L>(tab + o * RT, row);  // one row feeds both lines
    double Ex = 0.0, Fx = 0.0, Ey = 0.0, Fy = 0.0;
#pragma unroll
    for (int i = 0; i < HI; ++i) {
      Ex += row[i] * ex[i];
      Fx += row[HI + 1 + i] * fx[i];
      Ey += row[i] * ey[i];
      Fy += row[HI + 1 + i] * fy[i];
    }
    if constexpr (Q & 1) {
      Ex += row[HI] * mx;
      Ey += row[HI] * my;
    }
    dx[T::off(b, a, o)] = Ex + Fx;
    dy[T::off(b, o, a)] = Ey + Fy;
    if (Q - 1 - o != o) {
      dx[T::off(b, a, Q - 1 - o)] = Fx - Ex;
      dy[T::off(b, Q - 1 - o, a)] = Fy - Ey;
    }
  }
}

template <class T>
__global__ void __launch_bounds__(T::NT, T::MINB)
    op_line_kernel(const OpParams prm, const OpMats<T::P, T::Q> mats) {
  constexpr int P = T::P, Q = T::Q, NC = T::NC, QQ = T::QQ, Q3 = T::Q3;
  constexpr int EPB = T::EPB, NT = T::NT;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t qbar;
  __shared__ double red_scratch[NT / 32 + 1];
  if (prm.stop && *prm.stop) return;

  const int tid = threadIdx.x;
  const int slot = tid / QQ;
  const int l = tid - slot * QQ;
  const bool aslot = slot < EPB;
  double* S0 = smem + T::OFF_S + (aslot ? slot : 0) * 3 * T::SLAB;
  const double* sD = smem + T::OFF_D;
  const double* eBF = smem + T::OFF_EBF;
  const double* eBT = smem + T::OFF_EBT;
  const double* eDF = smem + T::OFF_EDF;
  const double* eDT = smem + T::OFF_EDT;
  for (int t = tid; t < Q * Q; t += NT) smem[T::OFF_D + (t / Q) * T::RQ + t % Q] = mats.D[t];
  // even-odd tables from the full matrices (op_eo.cuh)
  if constexpr (T::INTERP) {
    eo_build(smem + T::OFF_EBF, Q, P, [&](int o, int a) { return mats.B[o * P + a]; }, tid, NT);
    eo_build(smem + T::OFF_EBT, P, Q, [&](int o, int a) { return mats.B[a * P + o]; }, tid, NT);
  }
  eo_build(smem + T::OFF_EDF, Q, Q, [&](int o, int a) { return mats.D[o * Q + a]; }, tid, NT);
  eo_build(smem + T::OFF_EDT, Q, Q, [&](int o, int a) { return mats.D[a * Q + o]; }, tid, NT);
  __syncthreads();
  double* S1 = S0 + T::SLAB;
  double* S2 = S1 + T::SLAB;
  const int qa = l % Q, qb = l / Q;  // Q x Q line / column coordinates
  const int pa = l % P, pb = l / P;  // P x P line coordinates (l < P*P)
  // gather/scatter line of this thread: x-line (j = pa, k = pb) when
  // interpolating, z-column (i = qa, j = qb) when collocated
  const bool gthread = aslot && (T::INTERP ? l < P * P : (qa < P && qb < P));

  const int64_t nsteps = (prm.E + EPB - 1) / EPB;
  const int64_t G = gridDim.x;
  const int64_t NXY = prm.NX * prm.NY;

  const FastDiv divx((uint32_t)prm.nx), divy((uint32_t)prm.ny);
  // work slot -> element (a subset list for the partitioned overlap, else identity)
  auto elem_of = [&](int64_t k) -> int64_t { return prm.elist ? (int64_t)__ldg(prm.elist + k) : k; };
  auto geometry = [&](int64_t step) {
    LineGeo g{};
    const int64_t k = step * EPB + slot;
    g.active = gthread && step < nsteps && k < prm.E;
    if (!g.active) return g;
    const int64_t e = elem_of(k);
    const int li = T::INTERP ? 0 : qa, lj = T::INTERP ? pa : qb, lk = T::INTERP ? pb : 0;
    if (prm.idx) {
      g.tab = e * T::P3 + li + P * (lj + P * lk);
      g.tstep = T::INTERP ? 1 : P * P;
    } else {
      // element lattice position (E < 2^31: 32-bit fast division)
      const uint32_t e32 = (uint32_t)e, r = divx.div(e32), ez = divy.div(r);
      const uint32_t ex = e32 - r * (uint32_t)prm.nx, ey = r - ez * (uint32_t)prm.ny;
      const int64_t ix = (int64_t)ex * (P - 1) + li, iy = (int64_t)ey * (P - 1) + lj,
                    iz = (int64_t)ez * (P - 1) + lk;
      g.base = ix + prm.NX * iy + NXY * iz;
      g.step = T::INTERP ? 1 : NXY;
      if (prm.cons_mode == 1) {
        // on_bnd_face along the line: faces across the line take all of it,
        // the two faces it crosses take its first / last node
        const int f = prm.bnd_faces;
        const uint32_t all = (1u << P) - 1u;
        uint32_t cm = 0u;
        if (T::INTERP) {  // x-line
          if (((f & 4) && iy == 0) || ((f & 8) && iy == prm.NY - 1) || ((f & 16) && iz == 0) ||
              ((f & 32) && iz == prm.NZ - 1))
            cm = all;
          if ((f & 1) && ix == 0) cm |= 1u;
          if ((f & 2) && ix + P - 1 == prm.NX - 1) cm |= 1u << (P - 1);
        } else {  // z-line
          if (((f & 1) && ix == 0) || ((f & 2) && ix == prm.NX - 1) || ((f & 4) && iy == 0) ||
              ((f & 8) && iy == prm.NY - 1))
            cm = all;
          if ((f & 16) && iz == 0) cm |= 1u;
          if ((f & 32) && iz + P - 1 == prm.NZ - 1) cm |= 1u << (P - 1);
        }
        g.cmask = cm;
      }
    }
    if (prm.cons_mode == 2) {
#pragma unroll
      for (int n = 0; n < P; ++n) {
        const int64_t node = prm.idx ? (int64_t)prm.idx[g.tab + n * g.tstep] : g.base + n * g.step;
        g.cmask |= ((prm.cons_mask[node >> 5] >> (node & 31)) & 1u) << n;
      }
    }
    return g;
  };
  auto node_of = [&](const LineGeo& g, int n) -> int64_t {
    return prm.idx ? (int64_t)prm.idx[g.tab + n * g.tstep] : g.base + n * g.step;
  };
  auto load_line = [&](const LineGeo& g, int c, double* xn) {
    const double* xc = prm.x + c * prm.n_L;
#pragma unroll
    for (int n = 0; n < P; ++n) xn[n] = g.active ? __ldg(xc + node_of(g, n)) : 0.0;
  };

  // L2 prefetch of a step's geometric factors (bulk, no shared memory)
  auto prefetch_qd = [&](int64_t step) {
    if (step < nsteps) {
      const int64_t k0 = step * EPB;
      const int ne = (int)((prm.E - k0) < EPB ? (prm.E - k0) : EPB);
      if (prm.elist) {
        for (int i = 0; i < ne; ++i)
          bulk_prefetch_l2(prm.qd + elem_of(k0 + i) * T::QDS, (uint32_t)(T::QDS * 8));
      } else {
        bulk_prefetch_l2(prm.qd + k0 * T::QDS, (uint32_t)(ne * T::QDS * 8));
      }
    }
  };
  // staged factors (T::QS): one bulk copy per step into smem + OFF_QS
  auto issue_qs = [&](int64_t step) {
    const int64_t k0 = step * EPB;
    const int ne = (int)((prm.E - k0) < EPB ? (prm.E - k0) : EPB);
    mbar_arrive_expect_tx(&qbar, (uint32_t)(ne * T::QDS * 8));
    if (prm.elist) {
      for (int i = 0; i < ne; ++i)
        bulk_g2s(smem + T::OFF_QS + i * T::QDS, prm.qd + elem_of(k0 + i) * T::QDS,
                 (uint32_t)(T::QDS * 8), &qbar, l2_evict_first_policy());
    } else {
      bulk_g2s(smem + T::OFF_QS, prm.qd + k0 * T::QDS, (uint32_t)(ne * T::QDS * 8), &qbar,
               l2_evict_first_policy());
    }
  };
  if constexpr (T::QS) {
    if (tid == 0) {
      mbar_init(&qbar, 1);
      fence_mbar_init();
      if ((int64_t)blockIdx.x < nsteps) issue_qs(blockIdx.x);
    }
    __syncthreads();  // mbarrier init visible
  } else {
    if (tid == 0) prefetch_qd(blockIdx.x);
  }

  LineGeo gcur = geometry(blockIdx.x);
  double xn[P];
  load_line(gcur, 0, xn);

  double dot_acc = 0.0;
  int it = 0;
#pragma unroll 1
  for (int64_t step = blockIdx.x; step < nsteps; step += G, ++it) {
    const int64_t ks = step * EPB + slot;
    const bool eactive = aslot && ks < prm.E;
    const double* qd_el = T::QS ? smem + T::OFF_QS + (aslot ? slot : 0) * T::QDS
                                : prm.qd + (eactive ? elem_of(ks) : 0) * T::QDS;
    if (!T::QS && tid == 0) prefetch_qd(step + G);
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      double* yc = prm.y + c * prm.n_L;
      // masked input line of this item; the next item's raw line is loaded
      // below, after phase 3, to land while this one computes
      double u[P];
#pragma unroll
      for (int n = 0; n < P; ++n) u[n] = (gcur.active && !((gcur.cmask >> n) & 1u)) ? xn[n] : 0.0;

      double uq[Q];  // u at the quadrature points of this thread's column
      if constexpr (T::INTERP) {
        // ---- 1: x-interp of the gathered x-line -> S0 [k][j][qi] ----
        if (gthread) {
          double t[Q];
          eo_contract<P, Q, 1>(eBF, u, t);
          st_line<Q>(S0 + T::off(pb, pa, 0), t);
        }
        __syncthreads();
        // ---- 2: y-interp, line (qi, k) -> S1 [k][qj][qi] ----
        if (aslot && l < Q * P) {
          double ln[P], t[Q];
#pragma unroll
          for (int b = 0; b < P; ++b) ln[b] = S0[T::off(qb, b, qa)];
          eo_contract<P, Q, 1>(eBF, ln, t);
#pragma unroll
          for (int o = 0; o < Q; ++o) S1[T::off(qb, o, qa)] = t[o];
        }
        __syncthreads();
        // ---- 3: z-interp of the column (qi, qj) ----
        {
          double ln[P];
#pragma unroll
          for (int k = 0; k < P; ++k) ln[k] = aslot ? S1[T::off(k, qb, qa)] : 0.0;
          eo_contract<P, Q, 1>(eBF, ln, uq);
        }
      } else {
#pragma unroll
        for (int k = 0; k < Q; ++k) uq[k] = u[k < P ? k : 0];
      }
      // next item's raw line (geometry recomputed at the step end: fewer
      // registers live across the phases)
      if (c + 1 < NC) {
        load_line(gcur, c + 1, xn);
      } else {
        load_line(geometry(step + G), 0, xn);
      }

      double energy = 0.0;
      double w[Q];
      double g2[T::EARLY ? Q : 1];  // EARLY: z-derivative, then v2, of the column
      if constexpr (T::DIFF) {
        if (aslot) {
#pragma unroll
          for (int k = 0; k < Q; ++k) S2[T::off(k, qb, qa)] = uq[k];
        }
        if constexpr (T::EARLY) eo_contract<Q, Q, -1>(eDF, uq, g2);
        __syncthreads();
        // ---- 4: x and y derivatives, thread (a, b) = (qa, qb) ----
        if (aslot) {
          line_pair<T>(eDF, S2, S2, S0, S1, qa, qb);
        }
        __syncthreads();
        // ---- 5: z-derivative of the column (still in S2) + QFunction
        //      (qfunction.cpp:135-162); v2 replaces the column in S2 ----
        if constexpr (T::QS) {
          if (c == 0) mbar_wait(&qbar, (uint32_t)(it & 1));  // once per element step
        }
        if (aslot) {
          double ln[T::EARLY ? 1 : Q];
          if constexpr (!T::EARLY) {
#pragma unroll
            for (int k = 0; k < Q; ++k) ln[k] = S2[T::off(k, qb, qa)];
          }
          // (late form: partial unroll, two points' factors in flight)
#pragma unroll (T::EARLY ? Q : T::QFU)
          for (int k = 0; k < Q; ++k) {
            const int sp = T::off(k, qb, qa);
            const int pt = k * QQ + qb * Q + qa;
            double a2 = 0.0;  // z-derivative at point k
            if constexpr (T::EARLY) {
              a2 = g2[k];
            } else {  // row k of D . column
              double mrow[Q];
              line_row<Q>(sD + k * T::RQ, mrow);
#pragma unroll
              for (int c2 = 0; c2 < Q; ++c2) a2 += mrow[c2] * ln[c2];
            }
            const double a0 = S0[sp], a1 = S1[sp];
            double s00 = 0, s01 = 0, s02 = 0, s11 = 0, s12 = 0, s22 = 0;
            if (eactive) {
              if constexpr (T::QS) {
                s00 = qd_el[0 * Q3 + pt];
                s01 = qd_el[1 * Q3 + pt];
                s02 = qd_el[2 * Q3 + pt];
                s11 = qd_el[3 * Q3 + pt];
                s12 = qd_el[4 * Q3 + pt];
                s22 = qd_el[5 * Q3 + pt];
              } else {
                s00 = ld_stream(qd_el + 0 * Q3 + pt);
                s01 = ld_stream(qd_el + 1 * Q3 + pt);
                s02 = ld_stream(qd_el + 2 * Q3 + pt);
                s11 = ld_stream(qd_el + 3 * Q3 + pt);
                s12 = ld_stream(qd_el + 4 * Q3 + pt);
                s22 = ld_stream(qd_el + 5 * Q3 + pt);
              }
            }
            const double v0 = s00 * a0 + s01 * a1 + s02 * a2;
            const double v1 = s01 * a0 + s11 * a1 + s12 * a2;
            const double v2 = s02 * a0 + s12 * a1 + s22 * a2;
            S0[sp] = v0;
            S1[sp] = v1;
            if constexpr (T::EARLY)
              g2[k] = v2;
            else
              S2[sp] = v2;
            energy += a0 * v0 + a1 * v1 + a2 * v2;
          }
        }
        if constexpr (T::QS) {
          if (c == NC - 1) fence_proxy_async_smem();  // factor reads before the refill
        }
        __syncthreads();
        if constexpr (T::QS) {  // refill after the last component's QFunction
          if (c == NC - 1 && tid == 0 && step + G < nsteps) issue_qs(step + G);
        }
        // ---- 6: x^T and y^T derivatives in place ----
        if (aslot) {
          line_pair<T>(eDT, S0, S1, S0, S1, qa, qb);
        }
        __syncthreads();
        // ---- 7a: column sum with the z^T derivative ----
        {
          double ln[Q], t[Q];
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            if constexpr (T::EARLY)
              ln[k] = g2[k];
            else
              ln[k] = aslot ? S2[T::off(k, qb, qa)] : 0.0;
          }
          eo_contract<Q, Q, -1>(eDT, ln, t);
#pragma unroll
          for (int o = 0; o < Q; ++o) {
            const int sp = T::off(o, qb, qa);
            w[o] = aslot ? (S0[sp] + S1[sp] + t[o]) : 0.0;
          }
        }
      } else {
        // mass QFunction (qfunction.cpp:124-133), column-local
        if constexpr (T::QS) {
          if (c == 0) mbar_wait(&qbar, (uint32_t)(it & 1));
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const int pt = k * QQ + qb * Q + qa;
          const double m = eactive ? (T::QS ? qd_el[pt] : ld_stream(qd_el + pt)) : 0.0;
          w[k] = m * uq[k];
          energy += uq[k] * w[k];
        }
      }
      dot_acc += prm.coef * energy;

      if constexpr (T::INTERP) {
        // ---- 7b: z^T interp of the column -> S2 [c][qj][qi] ----
        if (aslot) {
          double t[P];
          eo_contract<Q, P, 1>(eBT, w, t);
#pragma unroll
          for (int k = 0; k < P; ++k) S2[T::off(k, qb, qa)] = t[k];
        }
        if constexpr (T::QS && !T::DIFF) {
          if (c == NC - 1) fence_proxy_async_smem();  // mass factor reads before the refill
        }
        __syncthreads();
        if constexpr (T::QS && !T::DIFF) {
          if (c == NC - 1 && tid == 0 && step + G < nsteps) issue_qs(step + G);
        }
        // ---- 8: y^T interp, line (qi, k) -> S1 [k][j][qi] ----
        if (aslot && l < Q * P) {
          double ln[Q], t[P];
#pragma unroll
          for (int o = 0; o < Q; ++o) ln[o] = S2[T::off(qb, o, qa)];
          eo_contract<Q, P, 1>(eBT, ln, t);
#pragma unroll
          for (int j = 0; j < P; ++j) S1[T::off(qb, j, qa)] = t[j];
        }
        __syncthreads();
        // ---- 9: x^T interp of the x-line (j, k), RED scatter ----
        if (gcur.active) {
          double ln[Q], t[P];
          ld_line<Q>(S1 + T::off(pb, pa, 0), ln);
          eo_contract<Q, P, 1>(eBT, ln, t);
#pragma unroll
          for (int i = 0; i < P; ++i)
            // constrained rows (y = x) are preset by the caller
            if (!((gcur.cmask >> i) & 1u) && !(prm.ablate & 2)) red_add(yc + node_of(gcur, i), prm.coef * t[i]);
        }
      } else {
        // collocated: the column thread scatters its z-line
        if (gcur.active) {
#pragma unroll
          for (int k = 0; k < P; ++k)
            if (!((gcur.cmask >> k) & 1u) && !(prm.ablate & 2)) red_add(yc + node_of(gcur, k), prm.coef * w[k]);
        }
      }
      // no trailing barrier: the next item's first shared-memory writes (S0 in
      // phase 1, S2 after phase 3) hit slabs whose last reads (phases 7a, 8)
      // are behind at least one barrier of this item; a column of S2 is only
      // ever rewritten by its own thread
    }
    gcur = geometry(step + G);
  }

  if (prm.dot_partials) {
    const double s = block_sum<NT>(dot_acc, red_scratch);
    if (tid == 0) prm.dot_partials[blockIdx.x] = s;
    pcg_alpha_epilogue<NT>(prm.fin, red_scratch);
  }
}

}  // namespace hxf
