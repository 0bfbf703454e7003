// K1 (line kernel): fused operator  y = G^T B^T D B G x  for the interpolating
// bases (BP1-BP4, q = p+2 Gauss points) and for the collocated sizes that have
// no tensor-core or pencil path (p >= 10).
//
// Every 1-D contraction is a register "line": one thread loads the Q (or P)
// values of one line of the element's slab, multiplies by the 1-D matrix whose
// entries are kernel-parameter constants (uniform, fully unrolled indices, so
// they are constant-bank operands of DFMA — no load per multiply-add) and
// writes the line back.  Phases (one __syncthreads between each):
//   1  x-interp  thread (j,k) gathers its node x-line straight from global
//      memory (software-pipelined one element ahead) -> S0 [k][j][qi]
//   2  y-interp  thread (qi,k)                        -> S1 [k][qj][qi]
//   3  z-interp  thread (qi,qj): u_q column in registers, -> S2, and the
//      z-derivative of it (registers)
//   4  x / y derivatives of S2 (thread (a,b) owns one x-line and one y-line)
//   5  QFunction per column, geometric factors loaded directly from global
//      memory (L2-prefetched one element ahead with cp.async.bulk.prefetch),
//      v0 / v1 in place, v2 in registers; p.(A p) as grad u . S grad u
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
#include "hxf_device.cuh"
#include "hxf_internal.h"
#include "op_kernel.cuh"
#include "pcg_device.cuh"

namespace hxf {

template <int P_, int Q_, int NC_, int QK_, bool INTERP_>
struct LineTraits {
  static constexpr int P = P_, Q = Q_, NC = NC_, QK = QK_;
  static constexpr bool INTERP = INTERP_;
  static constexpr bool DIFF = QK == 1;  // one qdata kind per launch (1 diffusion, 2 mass)
  static constexpr int QQ = Q * Q, Q3 = Q * Q * Q, P3 = P * P * P;
  static constexpr int EPB = QQ >= 64 ? 1 : (128 / QQ);
  static constexpr int NT = round_up(EPB * QQ, 32);
  static constexpr int MINB = (65536 / (NT * 128)) < 1 ? 1 : (65536 / (NT * 128) > 8 ? 8 : 65536 / (NT * 128));
  static constexpr int RS = Q | 1;        // odd row stride: x-line reads conflict-free
  static constexpr int SLAB = Q * Q * RS;
  static constexpr int NQD = DIFF ? 6 : 1;
  static constexpr int QDS = round_up(NQD * Q3, 2);  // padded doubles per element
  // 1-D matrices in shared memory, 16-byte rows (broadcast LDS.128 row loads):
  // B [Q][RP], B^T [P][RQ], D [Q][RQ], D^T [Q][RQ]
  static constexpr int RP = round_up(P, 2), RQ = round_up(Q, 2);
  static constexpr int OFF_B = 0, OFF_BT = Q * RP, OFF_D = OFF_BT + P * RQ, OFF_DT = OFF_D + Q * RQ;
  static constexpr int OFF_S = round_up(OFF_DT + Q * RQ, 2);
  static constexpr int SMEM_BYTES = (OFF_S + EPB * 3 * SLAB) * 8;
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

// N consecutive doubles of a 16-byte aligned shared-memory row into registers
template <int N>
__device__ __forceinline__ void line_row(const double* src, double* d) {
#pragma unroll
  for (int a = 0; a + 1 < N; a += 2) {
    const double2 v = *reinterpret_cast<const double2*>(src + a);
    d[a] = v.x;
    d[a + 1] = v.y;
  }
  if (N & 1) d[N - 1] = src[N - 1];
}

template <class T>
__global__ void __launch_bounds__(T::NT, T::MINB)
    op_line_kernel(const OpParams prm, const OpMats<T::P, T::Q> mats) {
  constexpr int P = T::P, Q = T::Q, NC = T::NC, QQ = T::QQ, Q3 = T::Q3;
  constexpr int EPB = T::EPB, NT = T::NT;
  extern __shared__ __align__(16) double smem[];
  __shared__ double red_scratch[NT / 32 + 1];
  if (prm.stop && *prm.stop) return;

  const int tid = threadIdx.x;
  const int slot = tid / QQ;
  const int l = tid - slot * QQ;
  const bool aslot = slot < EPB;
  double* S0 = smem + T::OFF_S + (aslot ? slot : 0) * 3 * T::SLAB;
  const double* sB = smem + T::OFF_B;
  const double* sBT = smem + T::OFF_BT;
  const double* sD = smem + T::OFF_D;
  const double* sDT = smem + T::OFF_DT;
  for (int t = tid; t < Q * Q; t += NT) {
    const int r = t / Q, c = t % Q;
    smem[T::OFF_D + r * T::RQ + c] = mats.D[t];
    smem[T::OFF_DT + c * T::RQ + r] = mats.D[t];
  }
  if constexpr (T::INTERP) {
    for (int t = tid; t < Q * P; t += NT) {
      const int r = t / P, c = t % P;  // B[r][c]
      smem[T::OFF_B + r * T::RP + c] = mats.B[t];
      smem[T::OFF_BT + c * T::RQ + r] = mats.B[t];
    }
  }
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

  auto geometry = [&](int64_t step) {
    LineGeo g{};
    const int64_t e = step * EPB + slot;
    g.active = gthread && step < nsteps && e < prm.E;
    if (!g.active) return g;
    const int li = T::INTERP ? 0 : qa, lj = T::INTERP ? pa : qb, lk = T::INTERP ? pb : 0;
    if (prm.idx) {
      g.tab = e * T::P3 + li + P * (lj + P * lk);
      g.tstep = T::INTERP ? 1 : P * P;
    } else {
      const int64_t ex = e % prm.nx, r = e / prm.nx, ey = r % prm.ny, ez = r / prm.ny;
      const int64_t ix = ex * (P - 1) + li, iy = ey * (P - 1) + lj, iz = ez * (P - 1) + lk;
      g.base = ix + prm.NX * iy + NXY * iz;
      g.step = T::INTERP ? 1 : NXY;
      if (prm.cons_mode == 1) {
#pragma unroll
        for (int n = 0; n < P; ++n) {
          const bool c = T::INTERP ? on_bnd_face(prm, ix + n, iy, iz) : on_bnd_face(prm, ix, iy, iz + n);
          if (c) g.cmask |= 1u << n;
        }
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
      const int64_t e0 = step * EPB;
      const int ne = (int)((prm.E - e0) < EPB ? (prm.E - e0) : EPB);
      bulk_prefetch_l2(prm.qd + e0 * T::QDS, (uint32_t)(ne * T::QDS * 8));
    }
  };
  if (tid == 0) prefetch_qd(blockIdx.x);

  LineGeo gcur = geometry(blockIdx.x);
  double xn[P];
  load_line(gcur, 0, xn);

  double dot_acc = 0.0;
#pragma unroll 1
  for (int64_t step = blockIdx.x; step < nsteps; step += G) {
    const int64_t e = step * EPB + slot;
    const bool eactive = aslot && e < prm.E;
    const double* qd_el = prm.qd + (eactive ? e : 0) * T::QDS;
    if (tid == 0) prefetch_qd(step + G);
    const LineGeo gnext = geometry(step + G);
#pragma unroll 1
    for (int c = 0; c < NC; ++c) {
      double* yc = prm.y + c * prm.n_L;
      // masked input line of this item; the next item's raw line is loaded
      // below, after phase 3, to land while this one computes
      double u[P];
#pragma unroll
      for (int n = 0; n < P; ++n) u[n] = (gcur.active && !((gcur.cmask >> n) & 1u)) ? xn[n] : 0.0;

      double uq[Q];  // u at the quadrature points of this thread's column
      double g2[Q];  // z-derivative of the column, then v2
      if constexpr (T::INTERP) {
        // ---- 1: x-interp of the gathered x-line ----
        if (gthread) {
#pragma unroll
          for (int o = 0; o < Q; ++o) {
            double mrow[P];
            line_row<P>(sB + o * T::RP, mrow);
            double s = 0.0;
#pragma unroll
            for (int a = 0; a < P; ++a) s += mrow[a] * u[a];
            S0[T::off(pb, pa, o)] = s;
          }
        }
        __syncthreads();
        // ---- 2: y-interp, line (qi, k) ----
        if (aslot && l < Q * P) {
          double ln[P];
#pragma unroll
          for (int b = 0; b < P; ++b) ln[b] = S0[T::off(qb, b, qa)];
#pragma unroll
          for (int o = 0; o < Q; ++o) {
            double mrow[P];
            line_row<P>(sB + o * T::RP, mrow);
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < P; ++b) s += mrow[b] * ln[b];
            S1[T::off(qb, o, qa)] = s;
          }
        }
        __syncthreads();
        // ---- 3: z-interp of the column (qi, qj) ----
        {
          double ln[P];
#pragma unroll
          for (int k = 0; k < P; ++k) ln[k] = aslot ? S1[T::off(k, qb, qa)] : 0.0;
#pragma unroll
          for (int o = 0; o < Q; ++o) {
            double mrow[P];
            line_row<P>(sB + o * T::RP, mrow);
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < P; ++k) s += mrow[k] * ln[k];
            uq[o] = s;
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < Q; ++k) uq[k] = u[k < P ? k : 0];
      }
      // next item's raw line
      {
        const LineGeo gn = c + 1 < NC ? gcur : gnext;
        load_line(gn, (c + 1) % NC, xn);
      }

      double energy = 0.0;
      double w[Q];
      if constexpr (T::DIFF) {
        if (aslot) {
#pragma unroll
          for (int k = 0; k < Q; ++k) S2[T::off(k, qb, qa)] = uq[k];
        }
#pragma unroll
        for (int o = 0; o < Q; ++o) {
          double mrow[Q];
          line_row<Q>(sD + o * T::RQ, mrow);
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < Q; ++k) s += mrow[k] * uq[k];
          g2[o] = s;
        }
        __syncthreads();
        // ---- 4: x and y derivatives, thread (a, b) = (qa, qb) ----
        if (aslot) {
          double lx[Q], ly[Q];
#pragma unroll
          for (int i = 0; i < Q; ++i) {
            lx[i] = S2[T::off(qb, qa, i)];
            ly[i] = S2[T::off(qb, i, qa)];
          }
#pragma unroll
          for (int o = 0; o < Q; ++o) {
            double mrow[Q];
            line_row<Q>(sD + o * T::RQ, mrow);  // one row feeds both lines
            double sx = 0.0, sy = 0.0;
#pragma unroll
            for (int i = 0; i < Q; ++i) {
              sx += mrow[i] * lx[i];
              sy += mrow[i] * ly[i];
            }
            S0[T::off(qb, qa, o)] = sx;
            S1[T::off(qb, o, qa)] = sy;
          }
        }
        __syncthreads();
        // ---- 5: QFunction on the column (qfunction.cpp:135-162) ----
        if (aslot) {
#pragma unroll
          for (int k = 0; k < Q; ++k) {
            const int sp = T::off(k, qb, qa);
            const int pt = k * QQ + qb * Q + qa;
            const double a0 = S0[sp], a1 = S1[sp], a2 = g2[k];
            double s00 = 0, s01 = 0, s02 = 0, s11 = 0, s12 = 0, s22 = 0;
            if (eactive) {
              s00 = ld_stream(qd_el + 0 * Q3 + pt);
              s01 = ld_stream(qd_el + 1 * Q3 + pt);
              s02 = ld_stream(qd_el + 2 * Q3 + pt);
              s11 = ld_stream(qd_el + 3 * Q3 + pt);
              s12 = ld_stream(qd_el + 4 * Q3 + pt);
              s22 = ld_stream(qd_el + 5 * Q3 + pt);
            }
            const double v0 = s00 * a0 + s01 * a1 + s02 * a2;
            const double v1 = s01 * a0 + s11 * a1 + s12 * a2;
            const double v2 = s02 * a0 + s12 * a1 + s22 * a2;
            S0[sp] = v0;
            S1[sp] = v1;
            g2[k] = v2;
            energy += a0 * v0 + a1 * v1 + a2 * v2;
          }
        }
        __syncthreads();
        // ---- 6: x^T and y^T derivatives in place ----
        if (aslot) {
          double lx[Q], ly[Q];
#pragma unroll
          for (int i = 0; i < Q; ++i) {
            lx[i] = S0[T::off(qb, qa, i)];
            ly[i] = S1[T::off(qb, i, qa)];
          }
#pragma unroll
          for (int o = 0; o < Q; ++o) {
            double mrow[Q];
            line_row<Q>(sDT + o * T::RQ, mrow);  // one row feeds both lines
            double sx = 0.0, sy = 0.0;
#pragma unroll
            for (int i = 0; i < Q; ++i) {
              sx += mrow[i] * lx[i];
              sy += mrow[i] * ly[i];
            }
            S0[T::off(qb, qa, o)] = sx;
            S1[T::off(qb, o, qa)] = sy;
          }
        }
        __syncthreads();
        // ---- 7a: column sum with the z^T derivative ----
#pragma unroll
        for (int o = 0; o < Q; ++o) {
          double mrow[Q];
          line_row<Q>(sDT + o * T::RQ, mrow);
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < Q; ++k) s += mrow[k] * g2[k];
          const int sp = T::off(o, qb, qa);
          w[o] = aslot ? (S0[sp] + S1[sp] + s) : 0.0;
        }
      } else {
        // mass QFunction (qfunction.cpp:124-133), column-local
#pragma unroll
        for (int k = 0; k < Q; ++k) {
          const int pt = k * QQ + qb * Q + qa;
          const double m = eactive ? ld_stream(qd_el + pt) : 0.0;
          w[k] = m * uq[k];
          energy += uq[k] * w[k];
        }
      }
      dot_acc += prm.coef * energy;

      if constexpr (T::INTERP) {
        // ---- 7b: z^T interp of the column -> S2 [c][qj][qi] ----
        if (aslot) {
#pragma unroll
          for (int k = 0; k < P; ++k) {
            double mrow[Q];
            line_row<Q>(sBT + k * T::RQ, mrow);
            double s = 0.0;
#pragma unroll
            for (int o = 0; o < Q; ++o) s += mrow[o] * w[o];
            S2[T::off(k, qb, qa)] = s;
          }
        }
        __syncthreads();
        // ---- 8: y^T interp, line (qi, k) -> S1 [k][j][qi] ----
        if (aslot && l < Q * P) {
          double ln[Q];
#pragma unroll
          for (int o = 0; o < Q; ++o) ln[o] = S2[T::off(qb, o, qa)];
#pragma unroll
          for (int j = 0; j < P; ++j) {
            double mrow[Q];
            line_row<Q>(sBT + j * T::RQ, mrow);
            double s = 0.0;
#pragma unroll
            for (int o = 0; o < Q; ++o) s += mrow[o] * ln[o];
            S1[T::off(qb, j, qa)] = s;
          }
        }
        __syncthreads();
        // ---- 9: x^T interp of the x-line (j, k), RED scatter ----
        if (gcur.active) {
          double ln[Q];
#pragma unroll
          for (int o = 0; o < Q; ++o) ln[o] = S1[T::off(pb, pa, o)];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double mrow[Q];
            line_row<Q>(sBT + i * T::RQ, mrow);
            double s = 0.0;
#pragma unroll
            for (int o = 0; o < Q; ++o) s += mrow[o] * ln[o];
            // constrained rows (y = x) are preset by the caller
            if (!((gcur.cmask >> i) & 1u) && !(prm.ablate & 2)) red_add(yc + node_of(gcur, i), prm.coef * s);
          }
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
      // are behind at least one barrier of this item
    }
    gcur = gnext;
  }

  if (prm.dot_partials) {
    const double s = block_sum<NT>(dot_acc, red_scratch);
    if (tid == 0) prm.dot_partials[blockIdx.x] = s;
    pcg_alpha_epilogue<NT>(prm.fin, red_scratch);
  }
}

}  // namespace hxf
