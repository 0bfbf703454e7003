// Microtest: TMA (cp.async.bulk.tensor) of an 8x8x8 f64 box out of a
// [m][NZ][NY][NX] lattice at an arbitrary (odd) start, for swizzle modes
// none / 64B / 128B; dumps the raw shared-memory image so the host can pin
// the layout formula the DMMA kernel reads with.  Also tries the instruction
// forms (with / without .tile, 3-D / 4-D, descriptor in param / global space).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int FORM>
__global__ void k(const __grid_constant__ CUtensorMap tm, const CUtensorMap* gtm, int x0, int y0,
                  int z0, int c, double* out) {
  __shared__ __align__(1024) double s[512];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(smem_u32(&bar)));
    if (FORM == 0)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(s)),
          "l"(&tm), "r"(x0), "r"(y0), "r"(z0), "r"(c), "r"(smem_u32(&bar))
          : "memory");
    if (FORM == 1)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(s)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(z0), "r"(c),
          "r"(smem_u32(&bar))
          : "memory");
    if (FORM == 2) {
      asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(gtm) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(s)),
          "l"(reinterpret_cast<uint64_t>(gtm)), "r"(x0), "r"(y0), "r"(z0), "r"(c),
          "r"(smem_u32(&bar))
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = s[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int NX = 16, NY = 12, NZ = 10, M = 2;
  const size_t n = size_t(NX) * NY * NZ * M;
  std::vector<double> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = double(i);
  double *d, *o;
  CUtensorMap* gtm;
  cudaMalloc(&d, n * 8);
  cudaMalloc(&o, 512 * 8);
  cudaMalloc(&gtm, sizeof(CUtensorMap));
  cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  printf("entry point: %s status %d fn %p; sizeof(CUtensorMap) %zu align %zu\n", cudaGetErrorString(ge),
         (int)q, fn, sizeof(CUtensorMap), alignof(CUtensorMap));
  if (!fn) return 1;
  const int modes[3] = {0, 64, 128};
  const CUtensorMapSwizzle sw[3] = {CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                    CU_TENSOR_MAP_SWIZZLE_128B};
  int fails = 0;
  for (int form = 0; form < 3; ++form) {
    if (only >= 0 && form != only) continue;
    for (int mi = 0; mi < 3; ++mi) {
      CUtensorMap tm;
      cuuint64_t dims[4] = {NX, NY, NZ, M};
      cuuint64_t strides[3] = {NX * 8ull, NX * NY * 8ull, NX * NY * NZ * 8ull};
      cuuint32_t box[4] = {8, 8, 8, 1};
      cuuint32_t es[4] = {1, 1, 1, 1};
      CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, d, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw[mi],
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("mode %d: encode failed %d\n", modes[mi], (int)r); ++fails; continue; }
      cudaMemcpy(gtm, &tm, sizeof tm, cudaMemcpyHostToDevice);
      const int x0 = 7, y0 = 3, z0 = 1, c = 1;
      if (form == 0) k<0><<<1, 128>>>(tm, gtm, x0, y0, z0, c, o);
      if (form == 1) k<1><<<1, 128>>>(tm, gtm, x0, y0, z0, c, o);
      if (form == 2) k<2><<<1, 128>>>(tm, gtm, x0, y0, z0, c, o);
      std::vector<double> s(512);
      cudaError_t e = cudaMemcpy(s.data(), o, 512 * 8, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("form %d mode %d: %s\n", form, modes[mi], cudaGetErrorString(e)); return 1; }
      int bad = 0;
      for (int kz = 0; kz < 8; ++kz)
        for (int j = 0; j < 8; ++j)
          for (int i = 0; i < 8; ++i) {
            uint32_t a = (kz * 512 + j * 64 + i * 8);
            if (modes[mi] == 64) a ^= ((a >> 7) & 3) << 4;
            if (modes[mi] == 128) a ^= ((a >> 7) & 7) << 4;
            const double want = double(((size_t(c) * NZ + z0 + kz) * NY + y0 + j) * NX + x0 + i);
            bad += s[a / 8] != want;
          }
      printf("form %d swizzle %3d: %d of 512 values off the formula (s[0]=%g s[1]=%g s[8]=%g)\n", form,
             modes[mi], bad, s[0], s[1], s[8]);
      fails += bad != 0;
    }
  }
  return fails ? 2 : 0;
}
