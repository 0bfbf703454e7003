// Instantiates the fused operator kernel for one degree P = p+1 (included by
// op_inst_p<P>.cu with HXF_P defined, so the instances compile in parallel).
#include <cmath>
#include <cstring>

#include "op_kernel.cuh"
#include "op_pencil.cuh"
#include "op_dmma.cuh"
#include "op_line.cuh"
#include "op_dmmaeo.cuh"
#include "op_dmma3.cuh"

namespace hxf {
namespace {

template <int P, int Q, int NC, bool INTERP, int QK>
struct Pick {
  // stream the geometric factors through shared memory (bulk copy, double
  // buffered) whenever that still leaves room for two CTAs per SM
  static constexpr bool QSMEM = OpTraits<P, Q, NC, INTERP, QK, true>::SMEM_BYTES <= 112 * 1024;
  using T = OpTraits<P, Q, NC, INTERP, QK, QSMEM>;
};

template <class T>
cudaError_t run(const OpParams& prm, const double* B, const double* D, cudaStream_t s,
                int* grid_out) {
  static int max_ctas = -1;
  auto kern = op_apply_kernel<T>;
  if (max_ctas < 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int nb = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::NT, T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (nb < 1) return cudaErrorInvalidConfiguration;
    max_ctas = nb * num_sms();
  }
  if (prm.elist) return cudaErrorNotSupported;  // no element-list support
  OpMats<T::P, T::Q> mats;
  std::memset(&mats, 0, sizeof mats);
  if (T::INTERP) std::memcpy(mats.B, B, sizeof(double) * T::Q * T::P);
  std::memcpy(mats.D, D, sizeof(double) * T::Q * T::Q);
  const int64_t nsteps = (prm.E + T::EPB - 1) / T::EPB;
  const int grid = capped_grid(nsteps, max_ctas);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  kern<<<grid, T::NT, T::SMEM_BYTES, s>>>(prm, mats);
  count_launch();
  return cudaGetLastError();
}

// The line kernel's even-odd contractions need centro-symmetric 1-D matrices
// (B[q-1-i][p-j] = B[i][j], D[q-1-i][q-1-j] = -D[i][j]: symmetric GLL nodes and
// Gauss / GLL points, make_basis, tensor_basis.cpp:40-71).  Anything else
// takes the general kernel.
// Line kernel (op_line.cuh): interpolating bases and the large collocated sizes.
template <class T>
cudaError_t run_line(const OpParams& prm, const double* B, const double* D, cudaStream_t s,
                     int* grid_out) {
  static int max_ctas = -1;
  auto kern = op_line_kernel<T>;
  if (max_ctas < 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int nb = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::NT, T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (nb < 1) return cudaErrorInvalidConfiguration;
    max_ctas = nb * num_sms();
  }
  OpMats<T::P, T::Q> mats;
  std::memset(&mats, 0, sizeof mats);
  if (T::INTERP) std::memcpy(mats.B, B, sizeof(double) * T::Q * T::P);
  std::memcpy(mats.D, D, sizeof(double) * T::Q * T::Q);
  const int64_t nsteps = (prm.E + T::EPB - 1) / T::EPB;
  const int grid = capped_grid(nsteps, max_ctas);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  kern<<<grid, T::NT, T::SMEM_BYTES, s>>>(prm, mats);
  count_launch();
  return cudaGetLastError();
}

// Collocated diffusion fast path (op_pencil.cuh) when its single-stage
// footprint leaves room for at least two CTAs per SM.
template <class T>
cudaError_t run_pencil(const OpParams& prm, const double* D, cudaStream_t s, int* grid_out) {
  static int max_ctas = -1;
  auto kern = op_pencil_kernel<T>;
  if (max_ctas < 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int nb = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::NT, T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (nb < 1) return cudaErrorInvalidConfiguration;
    max_ctas = nb * num_sms();
  }
  static_assert(T::GM == 0 || T::GM == 1, "gather mode");
  (void)D;
  if (!prm.D) return cudaErrorInvalidValue;
  const int64_t nsteps = (prm.E + T::EPB - 1) / T::EPB;
  const int grid = capped_grid(nsteps, max_ctas);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  kern<<<grid, T::NT, T::SMEM_BYTES, s>>>(prm);
  count_launch();
  return cudaGetLastError();
}

// p = 7 collocated diffusion on the FP64 tensor cores (op_dmma.cuh).
template <class T>
cudaError_t run_dmma(const OpParams& prm, cudaStream_t s, int* grid_out) {
  static int max_ctas = -1;
  auto kern = op_dmma_kernel<T>;
  if (max_ctas < 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int nb = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::NT, T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (nb < 1) return cudaErrorInvalidConfiguration;
    max_ctas = nb * num_sms();
  }
  if (!prm.D) return cudaErrorInvalidValue;
  const int grid = capped_grid(prm.E, max_ctas);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  CUtensorMap xmap;
  std::memset(&xmap, 0, sizeof xmap);
  if constexpr (T::TMA)
    if (!encode_lattice_map(prm, T::NC, &xmap)) return cudaErrorInvalidValue;
  const cudaError_t err = launch_pdl_if(pdl_enabled() || prm.pdl, kern, dim3(grid), dim3(T::NT),
                                        T::SMEM_BYTES, s, prm, xmap);
  count_launch();
  return err;
}

// p = 8..15 collocated diffusion, even-odd halves on the FP64 tensor cores
// (op_dmmaeo.cuh); structured box only (lattice gather).
template <class T>
cudaError_t run_dmmaeo(const OpParams& prm, cudaStream_t s, int* grid_out) {
  static int max_ctas = -1;
  auto kern = op_dmmaeo_kernel<T>;
  if (max_ctas < 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int nb = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::NT, T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (nb < 1) return cudaErrorInvalidConfiguration;
    max_ctas = nb * num_sms();
  }
  if (!prm.D || prm.idx || prm.cons_mode == 2) return cudaErrorInvalidValue;
  const int grid = capped_grid(prm.E, max_ctas);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  const cudaError_t err =
      launch_pdl_if(pdl_enabled() || prm.pdl, kern, dim3(grid), dim3(T::NT), T::SMEM_BYTES, s, prm);
  count_launch();
  return err;
}

// BP6 p = 6, 7: the three components batched through every phase (op_dmma3.cuh)
template <class T>
cudaError_t run_dmma3(const OpParams& prm, cudaStream_t s, int* grid_out) {
  static int max_ctas = -1;
  auto kern = op_dmma3_kernel<T>;
  if (max_ctas < 0) {
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    int nb = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, T::NT, T::SMEM_BYTES);
    if (err != cudaSuccess) return err;
    if (nb < 1) return cudaErrorInvalidConfiguration;
    max_ctas = nb * num_sms();
  }
  if (!prm.D) return cudaErrorInvalidValue;
  const int grid = capped_grid(prm.E, max_ctas);
  if (grid_out) *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  const cudaError_t err =
      launch_pdl_if(pdl_enabled() || prm.pdl, kern, dim3(grid), dim3(T::NT), T::SMEM_BYTES, s, prm);
  count_launch();
  return err;
}

template <int NP>
cudaError_t run_dmma3_gm(const OpParams& prm, cudaStream_t s, int* g) {
  if (!prm.idx && prm.cons_mode != 2) return run_dmma3<Dmma3Traits<0, NP>>(prm, s, g);
  return run_dmma3<Dmma3Traits<1, NP>>(prm, s, g);
}

template <int NC, int NW, int NP = 8>
cudaError_t run_dmma_nw(const OpParams& prm, cudaStream_t s, int* g) {
  if constexpr (NP == 8 && NW == 4) {
    if (dmma_stages() == 2) {
      if (!prm.idx && prm.cons_mode != 2) return run_dmma<DmmaTraits<NC, 0, NW, NP, 2>>(prm, s, g);
      return run_dmma<DmmaTraits<NC, 1, NW, NP, 2>>(prm, s, g);
    }
  }
  if (!prm.idx && prm.cons_mode != 2) {
    // structured box: the x slab by tensor-map TMA where the lattice allows it
    if constexpr (NW == 4)
      if (lattice_tma_ok(prm, NC)) return run_dmma<DmmaTraits<NC, 0, NW, NP, 1, true>>(prm, s, g);
    return run_dmma<DmmaTraits<NC, 0, NW, NP>>(prm, s, g);
  }
  return run_dmma<DmmaTraits<NC, 1, NW, NP>>(prm, s, g);
}

template <int NC, int NP = 8>
cudaError_t run_dmma_gm(const OpParams& prm, cudaStream_t s, int* g) {
  if constexpr (NP != 8) {
    return run_dmma_nw<NC, 4, NP>(prm, s, g);
  } else {
    switch (dmma_warps()) {
      case 8:
        return run_dmma_nw<NC, 8>(prm, s, g);
      case 2:
        return run_dmma_nw<NC, 2>(prm, s, g);
      default:
        return run_dmma_nw<NC, 4>(prm, s, g);
    }
  }
}

template <int P, int NC>
constexpr bool use_pencil() {
  return P <= 10 && PencilTraits<P, NC, 0>::SMEM_BYTES <= 112 * 1024;
}

template <int P, int NC>
cudaError_t run_pencil_gm(const OpParams& prm, const double* D, cudaStream_t s, int* g) {
  if (!prm.idx && prm.cons_mode != 2) return run_pencil<PencilTraits<P, NC, 0>>(prm, D, s, g);
  return run_pencil<PencilTraits<P, NC, 1>>(prm, D, s, g);
}

template <int P, int Q, bool INTERP>
cudaError_t run_q(int NC, int qk, const OpParams& prm, const double* B, const double* D,
                  cudaStream_t s, int* g) {
  if constexpr (!INTERP && P == 8) {
    // p = 7 collocated diffusion on the FP64 tensor cores
    if (qk == 1 && op_kernel_choice() == 0) {
      if (NC == 1) return run_dmma_gm<1>(prm, s, g);
      if (NC == 3 && dmma3_enabled()) return run_dmma3_gm<8>(prm, s, g);
      if (NC == 3) return run_dmma_gm<3>(prm, s, g);
    }
  }
  if constexpr (!INTERP && P >= 9 && P <= 16) {
    // high orders: even-odd halves on the FP64 tensor cores (structured box)
    if (qk == 1 && op_kernel_choice() == 0 && dmmaeo_enabled(P, NC) && !prm.idx &&
        prm.cons_mode != 2 && centro_symmetric(P, Q, false, B, D)) {
      if (NC == 1) return run_dmmaeo<EoTraits<P, 1>>(prm, s, g);
      if (NC == 3) return run_dmmaeo<EoTraits<P, 3>>(prm, s, g);
    }
  }
  if constexpr (!INTERP && P == 7) {
    // p = 6, three components: the zero-padded 8^3 tensor-core tile beats the
    // pencil kernel (C4 BP6 p=6 40^3: K1 833 vs 1098 us); one component and
    // p = 4, 5 do not (fixed 8^3 tile cost per element: p=4 BP5 753 vs 297 us)
    if (qk == 1 && NC == 3 && op_kernel_choice() == 0 && !dmma_pad_disabled())
      return dmma3_enabled() ? run_dmma3_gm<P>(prm, s, g) : run_dmma_gm<3, P>(prm, s, g);
  }
  if constexpr (!INTERP) {
    // three components: the pencil kernel (even-odd; ahead of the line kernel
    // for BP6 p = 2, 4, 5, 8, 9); one component: the line kernel wins at every p != 7
    // (BP5 1e7 DOFs, K1 roof line / pencil: p=1 0.55/0.48, p=3 0.76/0.54,
    // p=6 0.54/0.49, p=8 0.57/0.46, p=9 0.51/0.46, p=2,4,5 within 3 %)
    // (p = 3, 4: the line kernel, K1 263 vs 350 and 257 vs 283 us at 1e7 DOFs)
    if (qk == 1 && NC == 3 && P != 4 && P != 5 && use_pencil<P, 3>() && !pencil_disabled() &&
        centro_symmetric(P, Q, false, B, D))
      return run_pencil_gm<P, 3>(prm, D, s, g);
  }
  if (op_kernel_choice() != 2 && centro_symmetric(P, Q, INTERP, B, D)) {
    if (NC == 1 && qk == 1) return run_line<LineTraits<P, Q, 1, 1, INTERP>>(prm, B, D, s, g);
    if (NC == 1 && qk == 2) return run_line<LineTraits<P, Q, 1, 2, INTERP>>(prm, B, D, s, g);
    if (NC == 3 && qk == 1) return run_line<LineTraits<P, Q, 3, 1, INTERP>>(prm, B, D, s, g);
    if (NC == 3 && qk == 2) return run_line<LineTraits<P, Q, 3, 2, INTERP>>(prm, B, D, s, g);
  }
  if (NC == 1 && qk == 1) return run<typename Pick<P, Q, 1, INTERP, 1>::T>(prm, B, D, s, g);
  if (NC == 1 && qk == 2) return run<typename Pick<P, Q, 1, INTERP, 2>::T>(prm, B, D, s, g);
  if (NC == 3 && qk == 1) return run<typename Pick<P, Q, 3, INTERP, 1>::T>(prm, B, D, s, g);
  if (NC == 3 && qk == 2) return run<typename Pick<P, Q, 3, INTERP, 2>::T>(prm, B, D, s, g);
  return cudaErrorNotSupported;
}

}  // namespace

#define HXF_CAT2(a, b) a##b
#define HXF_CAT(a, b) HXF_CAT2(a, b)
cudaError_t HXF_CAT(launch_op_p, HXF_P)(int Q, int NC, bool interp, int qk, const OpParams& prm,
                                       const double* B, const double* D, cudaStream_t s,
                                       int* grid_out) {
  constexpr int P = HXF_P;
  if (!interp && Q == P) return run_q<P, P, false>(NC, qk, prm, B, D, s, grid_out);
  if (interp && Q == P + 1) return run_q<P, P + 1, true>(NC, qk, prm, B, D, s, grid_out);
  return cudaErrorNotSupported;
}

}  // namespace hxf
