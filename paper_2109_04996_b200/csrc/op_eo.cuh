// Even-odd ("centro-symmetric") 1-D contractions shared by the line and
// pencil operator kernels.  On symmetric GLL nodes with Gauss / GLL points the
// 1-D matrices satisfy M[NO-1-o][NI-1-a] = S M[o][a] (S = +1 interpolation,
// -1 derivative), so out = M in costs half the multiply-adds from a half-size
// table: row o < ceil(NO/2) = [ (M[o][a] + M[o][a'])/2 for a < NI/2 | M[o][NI/2]
// (odd NI, else 0) | (M[o][a] - M[o][a'])/2 for a < NI/2 ], a' = NI-1-a,
// 16-byte aligned rows of eo_row_stride(NI) doubles.
#pragma once
#include "hxf_device.cuh"

namespace hxf {

__host__ __device__ constexpr int eo_row_stride(int ni) { return (2 * (ni / 2) + 1 + 1) / 2 * 2; }
__host__ __device__ constexpr int eo_table_size(int no, int ni) { return ((no + 1) / 2) * eo_row_stride(ni); }

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

// Even-odd ("centro-symmetric") contraction: out[o] = sum_a M[o][a] in[a] for a
// NO x NI matrix with M[NO-1-o][NI-1-a] = S M[o][a] (S = +1 interpolation,
// -1 derivative on symmetric GLL / Gauss points), from the half-size table of
// LineTraits (one row per output pair): half the multiply-adds and row loads.
template <int NI, int NO, int S>
__device__ __forceinline__ void eo_contract(const double* tab, const double* in, double* out) {
  constexpr int HI = NI / 2, HO = (NO + 1) / 2, L = 2 * HI + 1, RT = (L + 1) / 2 * 2;
  double e[HI > 0 ? HI : 1], f[HI > 0 ? HI : 1];
#pragma unroll
  for (int a = 0; a < HI; ++a) {
    e[a] = in[a] + in[NI - 1 - a];
    f[a] = in[a] - in[NI - 1 - a];
  }
#pragma unroll
  for (int o = 0; o < HO; ++o) {
    double row[L];
    line_row<L>(tab + o * RT, row);
    double E = 0.0, F = 0.0;
#pragma unroll
    for (int a = 0; a < HI; ++a) {
      E += row[a] * e[a];
      F += row[HI + 1 + a] * f[a];
    }
    if constexpr (NI & 1) E += row[HI] * in[HI];
    out[o] = E + F;
    if (NO - 1 - o != o) out[NO - 1 - o] = S > 0 ? E - F : F - E;
  }
}

// Two lines through the same table (one broadcast row load per output pair).
template <int N, int S>
__device__ __forceinline__ void eo_pair(const double* tab, const double* in1, const double* in2,
                                        double* out1, double* out2) {
  constexpr int HI = N / 2, HO = (N + 1) / 2, L = 2 * HI + 1, RT = (L + 1) / 2 * 2;
  double e1[HI > 0 ? HI : 1], f1[HI > 0 ? HI : 1], e2[HI > 0 ? HI : 1], f2[HI > 0 ? HI : 1];
#pragma unroll
  for (int a = 0; a < HI; ++a) {
    e1[a] = in1[a] + in1[N - 1 - a];
    f1[a] = in1[a] - in1[N - 1 - a];
    e2[a] = in2[a] + in2[N - 1 - a];
    f2[a] = in2[a] - in2[N - 1 - a];
  }
#pragma unroll
  for (int o = 0; o < HO; ++o) {
    double row[L];
    line_row<L>(tab + o * RT, row);
    double E1 = 0.0, F1 = 0.0, E2 = 0.0, F2 = 0.0;
#pragma unroll
    for (int a = 0; a < HI; ++a) {
      E1 += row[a] * e1[a];
      F1 += row[HI + 1 + a] * f1[a];
      E2 += row[a] * e2[a];
      F2 += row[HI + 1 + a] * f2[a];
    }
    if constexpr (N & 1) {
      E1 += row[HI] * in1[HI];
      E2 += row[HI] * in2[HI];
    }
    out1[o] = E1 + F1;
    out2[o] = E2 + F2;
    if (N - 1 - o != o) {
      out1[N - 1 - o] = S > 0 ? E1 - F1 : F1 - E1;
      out2[N - 1 - o] = S > 0 ? E2 - F2 : F2 - E2;
    }
  }
}

// Build the table of an NO x NI matrix given by the accessor M(o, a) into
// shared memory (all threads of the CTA, stride nt).
template <class F>
__device__ __forceinline__ void eo_build(double* dst, int NO, int NI, F M, int tid, int nt) {
  const int HI = NI / 2, RT = eo_row_stride(NI), HO = (NO + 1) / 2;
  for (int t = tid; t < HO * RT; t += nt) {
    const int o = t / RT, c = t % RT;
    double v = 0.0;
    if (c < HI)
      v = 0.5 * (M(o, c) + M(o, NI - 1 - c));
    else if (c == HI)
      v = (NI & 1) ? M(o, HI) : 0.0;
    else if (c < 2 * HI + 1)
      v = 0.5 * (M(o, c - HI - 1) - M(o, NI - 1 - (c - HI - 1)));
    dst[t] = v;
  }
}

}  // namespace hxf
