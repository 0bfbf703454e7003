// K1 (collocated BP5/BP6 fast path): pencil-decomposed fused operator
//   y = G^T D^T S D G x   on GLL-collocated elements (interp1d == I).
//
// Same contract as op_apply_kernel (op_kernel.cuh) — masked gather, RED
// scatter, constrained y = x, fused p.Ap partials — restructured for the
// sm_100a memory system.  Per work item (element, component) four phases,
// one __syncthreads each, every 1-D contraction a register "pencil":
//   F  thread (a,b) reads the x-line (j=a,k=b) and the y-line (i=a,k=b) of
//      the gathered slab A and applies D to both, one D row (broadcast from
//      shared memory) feeding two pencils: g0 -> slab C, g1 -> slab B;
//   P  thread (i,j) re-reads its z-line of A, writes the NEXT item's masked
//      z-line into A (software-pipelined gather: its global loads were issued
//      one item earlier), applies D along z in registers and the pointwise
//      QFunction with the geometric factors from shared memory; v0 -> C,
//      v1 -> B in place; p.(A p) accumulates as grad u . S grad u;
//   T  thread (a,b) applies D^T to its x-line of C and y-line of B, in place;
//   Z  thread (i,j) applies D^T along z, sums, and scatters with FP64 RED.
// Slab rows are XOR-rotated in 16-byte chunks for p = 7 (padded otherwise)
// and planes skewed by half a bank cycle, so every shared access is
// conflict-free.  The element's geometric factors (6 P^3 doubles) arrive by
// one bulk async copy (TMA engine, L2 evict_first) issued as soon as phase P
// of the previous element has consumed its factors.
// Reference semantics: proj/src/operator.cpp:64-144 (see op_kernel.cuh).
#pragma once
#include "hxf_device.cuh"
#include "hxf_internal.h"
#include "op_eo.cuh"
#include "pcg_device.cuh"

namespace hxf {

__host__ __device__ constexpr int pencil_round_up(int a, int b) { return (a + b - 1) / b * b; }
__host__ __device__ constexpr int pencil_row_stride(int P) {
  // smallest RS >= P with RS = 2 (mod 4): 16-byte aligned rows whose 8-lane
  // LDS.128 phases fall on distinct bank quads
  return ((P + 1) / 4) * 4 + 2 >= P ? ((P + 1) / 4) * 4 + 2 : ((P + 1) / 4) * 4 + 6;
}

template <int P_, int NC_, int GM_>
struct PencilTraits {
  // GM 0: structured box, constraints none/box boundary (lattice-computed G);
  // GM 1: general — int32 index table and/or constraint bitmask.
  static constexpr int P = P_, NC = NC_, GM = GM_, PP = P * P, P3 = P * P * P;
  static constexpr int EPB = PP >= 64 ? 1 : (PP == 25 ? 5 : (PP == 36 ? 3 : (PP == 49 ? 2 : 64 / PP)));
  static constexpr int NT = pencil_round_up(EPB * PP, 32);
  static constexpr bool SWZ = (P == 8);  // XOR-rotated 64-byte rows
  // p != 7: layout searched for the fewest shared-memory wavefronts over the
  // kernel's three access patterns (x-line rows, y-columns, z-lines; scalar
  // 8-byte accesses, 34 % bank conflicts with the 16-byte aligned layout at
  // p = 8): RS = P and a plane stride PL_SEARCH; other P keep the aligned rows
  static constexpr int PL_SEARCH = P == 6 ? 37 : (P == 9 ? 81 : 0);  // (P = 10: measured +2.5 %)
  static constexpr bool VROW = SWZ || PL_SEARCH == 0;  // 16-byte row chunks (LDS.128)
  static constexpr int RS = SWZ ? 8 : (VROW ? pencil_row_stride(P) : P);
  // plane stride: padded layouts skew consecutive planes by 16 banks (+64 B);
  // the swizzled p = 7 layout flips the row parity per plane instead (no pad)
  static constexpr int PL = SWZ ? P * RS : (VROW ? P * RS + 8 : PL_SEARCH);
  static constexpr int SLAB = P * PL;    // doubles per element slab
  static constexpr int QDS = 6 * P3;     // geometric factors per element (even)
  static constexpr int DR = pencil_round_up(P, 2);  // matrix row stride (16-byte rows)
  // D^T rows in shared memory too, except for p = 7 where the 512 B are what
  // it takes to fit 6 CTAs per SM (transposed rows read as D columns there)
  // even-odd tables of D and D^T (op_eo.cuh; the bases are centro-symmetric)
  static constexpr int OFF_D = 0, OFF_DT = eo_table_size(P, P);
  static constexpr int OFF_QD = pencil_round_up(2 * eo_table_size(P, P), 2);
  static constexpr int OFF_A = OFF_QD + EPB * QDS;
  static constexpr int OFF_B = OFF_A + EPB * SLAB;
  static constexpr int OFF_C = OFF_B + EPB * SLAB;
  static constexpr int SMEM_BYTES = (OFF_C + EPB * SLAB) * 8;

  // slab offset of point (i, j, k) — x index i, y index j, plane k
  __device__ static __forceinline__ int off(int k, int j, int i) {
    if constexpr (SWZ) {
      const int R = j ^ (k & 1);  // physical row: parity flips plane to plane
      return k * PL + R * RS + 2 * (((i >> 1) + (R >> 1)) & 3) + (i & 1);
    }
    return k * PL + j * RS + i;
  }
  // slab offset of the 16-byte chunk holding x indices (2c, 2c+1) of row (j, k)
  __device__ static __forceinline__ int chunk(int k, int j, int c) {
    if constexpr (SWZ) {
      const int R = j ^ (k & 1);
      return k * PL + R * RS + 2 * ((c + (R >> 1)) & 3);
    }
    return k * PL + j * RS + 2 * c;
  }
};

// Lattice placement of one (element, lane) work item: the z-line's first
// node (or the element id in table mode) and which of its P nodes are
// constrained (bit k).
struct PencilGeo {
  int64_t key;     // node of (i, j, k = 0) (structured box) or element id (table)
  uint32_t cmask;  // bit k: node k of the z-line is constrained
  bool active;
};

template <int P>
__device__ __forceinline__ void load_row(const double* src, double* dst) {
#pragma unroll
  for (int a = 0; a + 1 < P; a += 2) {
    const double2 v = *reinterpret_cast<const double2*>(src + a);
    dst[a] = v.x;
    dst[a + 1] = v.y;
  }
  if (P & 1) dst[P - 1] = src[P - 1];
}

template <class T>
__global__ void __launch_bounds__(T::NT) op_pencil_kernel(const OpParams prm) {
  constexpr int P = T::P, PP = T::PP, P3 = T::P3, EPB = T::EPB, NT = T::NT, NC = T::NC;
  extern __shared__ __align__(16) double smem[];
  __shared__ __align__(8) uint64_t qbar;
  __shared__ double red_scratch[NT / 32 + 1];
  if (prm.stop && *prm.stop) return;

  const int tid = threadIdx.x;
  const int slot = tid / PP;
  const int l = tid - slot * PP;
  const bool active_slot = slot < EPB;
  const int la = l % P, lb = l / P;  // (i,j) | (j,k) | (i,k) depending on the phase
  const double* eD = smem + T::OFF_D;    // even-odd D
  const double* eDT = smem + T::OFF_DT;  // even-odd D^T
  double* sQD = smem + T::OFF_QD;
  double* SA = smem + T::OFF_A + (active_slot ? slot : 0) * T::SLAB;
  double* SB = smem + T::OFF_B + (active_slot ? slot : 0) * T::SLAB;
  double* SC = smem + T::OFF_C + (active_slot ? slot : 0) * T::SLAB;
  const double* qd_el = sQD + (active_slot ? slot : 0) * T::QDS;

  eo_build(smem + T::OFF_D, P, P, [&](int o, int a) { return prm.D[o * P + a]; }, tid, NT);
  eo_build(smem + T::OFF_DT, P, P, [&](int o, int a) { return prm.D[a * P + o]; }, tid, NT);

  const int64_t nsteps = (prm.E + EPB - 1) / EPB;
  const int64_t G = gridDim.x;
  const int64_t NXY = prm.NX * prm.NY;
  uint64_t policy = 0;
  // element of list position k: a subset (partition overlap: boundary
  // elements first, then the interior) or 0..E-1
  auto elem_of = [&](int64_t k) -> int64_t { return prm.elist ? (int64_t)__ldg(prm.elist + k) : k; };
  auto qbytes = [&](int64_t s) -> uint32_t {
    const int64_t e0 = s * EPB;
    const int ne = (int)((prm.E - e0) < EPB ? (prm.E - e0) : EPB);
    return (uint32_t)(ne * T::QDS * 8);
  };
  auto issue_qdata = [&](int64_t s) {
    const uint32_t bytes = qbytes(s);
    mbar_arrive_expect_tx(&qbar, bytes);
    if (prm.elist) {  // listed elements are not contiguous: one copy each
      const int ne = (int)(bytes / (T::QDS * 8));
      for (int i = 0; i < ne; ++i)
        bulk_g2s(sQD + i * T::QDS, prm.qd + elem_of(s * EPB + i) * T::QDS, (uint32_t)(T::QDS * 8),
                 &qbar, policy);
    } else {
      bulk_g2s(sQD, prm.qd + s * EPB * T::QDS, bytes, &qbar, policy);
    }
  };
  // the element after next: pull its factors HBM -> L2 now (no shared memory
  // needed), so the later bulk copy into shared memory is an L2 hit
  auto prefetch_qdata = [&](int64_t s) {
    if (s < nsteps && (prm.ablate & 8) && !prm.elist)
      bulk_prefetch_l2(prm.qd + s * EPB * T::QDS, qbytes(s));
  };
  if (tid == 0) {
    mbar_init(&qbar, 1);
    fence_mbar_init();
    policy = l2_evict_first_policy();
    if ((int64_t)blockIdx.x < nsteps && !(prm.ablate & 4)) issue_qdata(blockIdx.x);
    prefetch_qdata(blockIdx.x + G);
  }

  auto node_of = [&](const PencilGeo& g, int k) -> int64_t {
    if constexpr (T::GM == 0) return g.key + k * NXY;
    return prm.idx ? (int64_t)prm.idx[g.key * P3 + la + P * (lb + P * k)] : g.key + k * NXY;
  };
  const FastDiv divx((uint32_t)prm.nx), divy((uint32_t)prm.ny);
  auto geometry = [&](int64_t step) {
    PencilGeo g{};
    const int64_t k = step * EPB + slot;
    g.active = active_slot && step < nsteps && k < prm.E;
    if (!g.active) return g;
    const int64_t e = elem_of(k);
    if (T::GM == 1 && prm.idx) {
      g.key = e;
    } else {
      // element lattice position (E < 2^31: 32-bit fast division)
      const uint32_t e32 = (uint32_t)e, r = divx.div(e32), ez = divy.div(r);
      const uint32_t ex = e32 - r * (uint32_t)prm.nx, ey = r - ez * (uint32_t)prm.ny;
      const int64_t ix = (int64_t)ex * (P - 1) + la, iy = (int64_t)ey * (P - 1) + lb,
                    iz = (int64_t)ez * (P - 1);
      g.key = ix + prm.NX * iy + NXY * iz;
      if (T::GM == 0 && prm.cons_mode == 1) {
        // on_bnd_face along the z-line: x / y faces take the whole line
        const int f = prm.bnd_faces;
        const bool side = ((f & 1) && ix == 0) || ((f & 2) && ix == prm.NX - 1) ||
                          ((f & 4) && iy == 0) || ((f & 8) && iy == prm.NY - 1);
        uint32_t cm = side ? (1u << P) - 1u : 0u;
        if ((f & 16) && iz == 0) cm |= 1u;
        if ((f & 32) && iz + P - 1 == prm.NZ - 1) cm |= 1u << (P - 1);
        g.cmask = cm;
      }
    }
    if (T::GM == 1 && prm.cons_mode == 2) {
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const int64_t node = node_of(g, k);
        g.cmask |= ((prm.cons_mask[node >> 5] >> (node & 31)) & 1u) << k;
      }
    }
    return g;
  };
  // Work item q (0, 1, 2, ... for this CTA) = (element step, component).
  auto item_step = [&](int q) -> int64_t { return (int64_t)blockIdx.x + (int64_t)(q / NC) * G; };
  // raw (unmasked) z-line loads of work item (g, component c) into xn[]
  auto load_line = [&](const PencilGeo& g, int c, double* xn) {
#pragma unroll
    for (int k = 0; k < P; ++k)
      xn[k] = (g.active && !(prm.ablate & 1)) ? __ldg(prm.x + c * prm.n_L + node_of(g, k)) : 1.0;
  };
  auto store_line = [&](const PencilGeo& g, const double* xn) {
    if (!active_slot) return;
#pragma unroll
    for (int k = 0; k < P; ++k)
      SA[T::off(k, lb, la)] = (g.active && !((g.cmask >> k) & 1u)) ? xn[k] : 0.0;
  };

  // prologue: item 0 into slab A, item 1's loads in flight
  PencilGeo gcur = geometry(blockIdx.x);
  double xn[P];
  load_line(gcur, 0, xn);
  store_line(gcur, xn);
  PencilGeo gpf = NC > 1 ? gcur : geometry(item_step(1));  // geometry of the prefetched item
  load_line(gpf, 1 % NC, xn);
  __syncthreads();  // mbarrier init, matrices and slab A visible

  double dot_acc = 0.0;
  int it = 0, q = 0;
#pragma unroll 1
  for (int64_t step = blockIdx.x; step < nsteps; step += G, ++it) {
#pragma unroll 1
    for (int c = 0; c < NC; ++c, ++q) {
      double* yc = prm.y + c * prm.n_L;

      // ---- F: D along x (-> C) and y (-> B) from slab A, one D row per two pencils ----
      if (active_slot) {
        double row[P], col[P];
        if constexpr (T::VROW) {
#pragma unroll
          for (int a = 0; a + 1 < P; a += 2) {
            const double2 v = *reinterpret_cast<const double2*>(SA + T::chunk(lb, la, a / 2));
            row[a] = v.x;
            row[a + 1] = v.y;
          }
          if (P & 1) row[P - 1] = SA[T::off(lb, la, P - 1)];
        } else {
#pragma unroll
          for (int a = 0; a < P; ++a) row[a] = SA[T::off(lb, la, a)];
        }
#pragma unroll
        for (int b = 0; b < P; ++b) col[b] = SA[T::off(lb, b, la)];
        double gx[P], gy[P];
        eo_pair<P, -1>(eD, row, col, gx, gy);
#pragma unroll
        for (int o = 0; o < P; ++o) SB[T::off(lb, o, la)] = gy[o];
        if constexpr (T::VROW) {
#pragma unroll
          for (int a = 0; a + 1 < P; a += 2)
            *reinterpret_cast<double2*>(SC + T::chunk(lb, la, a / 2)) = make_double2(gx[a], gx[a + 1]);
          if (P & 1) SC[T::off(lb, la, P - 1)] = gx[P - 1];
        } else {
#pragma unroll
          for (int a = 0; a < P; ++a) SC[T::off(lb, la, a)] = gx[a];
        }
      }
      if (c == 0 && !(prm.ablate & 4)) mbar_wait(&qbar, (uint32_t)(it & 1));
      __syncthreads();

      // ---- P: z-line of A, next item's gather into A, D along z + QFunction ----
      double u[P];
#pragma unroll
      for (int k = 0; k < P; ++k) u[k] = active_slot ? SA[T::off(k, lb, la)] : 0.0;
      store_line(gpf, xn);  // item q+1's masked z-line (this thread's column only)
      gpf = ((q + 2) / NC == (q + 1) / NC && NC > 1) ? gpf : geometry(item_step(q + 2));
      load_line(gpf, (q + 2) % NC, xn);  // item q+2 lands while items q, q+1 compute
      double v2[P];
      double energy = 0.0;
      double g2v[P];
      eo_contract<P, P, -1>(eD, u, g2v);
#pragma unroll
      for (int k = 0; k < P; ++k) {
        const double g2 = g2v[k];
        const int sp = T::off(k, lb, la);
        const int pt = k * PP + lb * P + la;
        // (threads beyond the element slots read nothing: no race with the
        // active threads' in-place writes below)
        const double g0 = active_slot ? SC[sp] : 0.0, g1 = active_slot ? SB[sp] : 0.0;
        double s00 = 0, s01 = 0, s02 = 0, s11 = 0, s12 = 0, s22 = 0;
        if (gcur.active) {
          s00 = qd_el[0 * P3 + pt];
          s01 = qd_el[1 * P3 + pt];
          s02 = qd_el[2 * P3 + pt];
          s11 = qd_el[3 * P3 + pt];
          s12 = qd_el[4 * P3 + pt];
          s22 = qd_el[5 * P3 + pt];
        }
        const double v0 = s00 * g0 + s01 * g1 + s02 * g2;
        const double v1 = s01 * g0 + s11 * g1 + s12 * g2;
        v2[k] = s02 * g0 + s12 * g1 + s22 * g2;
        if (active_slot) {
          SC[sp] = v0;
          SB[sp] = v1;
        }
        // p.(A p) over free nodes = sum_e u_e^T A_e u_e = sum_points grad u . S grad u
        energy += g0 * v0 + g1 * v1 + g2 * v2[k];
      }
      dot_acc += prm.coef * energy;
      if (c == NC - 1) fence_proxy_async_smem();  // generic reads of the factors before the refill
      __syncthreads();
      // factors consumed: stream the next element's in while we finish this one
      if (c == NC - 1 && tid == 0 && step + G < nsteps && !(prm.ablate & 4)) {
        issue_qdata(step + G);
        prefetch_qdata(step + 2 * G);
      }

      // ---- T: D^T along x (C, in place) and y (B, in place) ----
      if (active_slot) {
        double row[P], col[P];
        if constexpr (T::VROW) {
#pragma unroll
          for (int a = 0; a + 1 < P; a += 2) {
            const double2 v = *reinterpret_cast<const double2*>(SC + T::chunk(lb, la, a / 2));
            row[a] = v.x;
            row[a + 1] = v.y;
          }
          if (P & 1) row[P - 1] = SC[T::off(lb, la, P - 1)];
        } else {
#pragma unroll
          for (int a = 0; a < P; ++a) row[a] = SC[T::off(lb, la, a)];
        }
#pragma unroll
        for (int b = 0; b < P; ++b) col[b] = SB[T::off(lb, b, la)];
        double tx[P], ty[P];
        eo_pair<P, -1>(eDT, row, col, tx, ty);
#pragma unroll
        for (int o = 0; o < P; ++o) SB[T::off(lb, o, la)] = ty[o];
        if constexpr (T::VROW) {
#pragma unroll
          for (int a = 0; a + 1 < P; a += 2)
            *reinterpret_cast<double2*>(SC + T::chunk(lb, la, a / 2)) = make_double2(tx[a], tx[a + 1]);
          if (P & 1) SC[T::off(lb, la, P - 1)] = tx[P - 1];
        } else {
#pragma unroll
          for (int a = 0; a < P; ++a) SC[T::off(lb, la, a)] = tx[a];
        }
      }
      __syncthreads();

      // ---- Z: D^T along z from registers + combine, G^T scatter ----
      if (gcur.active) {
        double zt[P];
        eo_contract<P, P, -1>(eDT, v2, zt);
#pragma unroll
        for (int k = 0; k < P; ++k) {
          const double s = zt[k];
          const int sp = T::off(k, lb, la);
          const double yk = prm.coef * (SC[sp] + SB[sp] + s);
          const int64_t node = node_of(gcur, k);
          // constrained rows (y = x) are preset by the caller
          if (!(prm.ablate & 2) && !((gcur.cmask >> k) & 1u)) red_add(yc + node, yk);
        }
      }
      __syncthreads();  // B and C free for the next item's phase F
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
