// Microtest: minimal 2-D TMA load (f64, 8x8 box) — which descriptor
// placement works on this driver / GPU:
//   v0 param (__grid_constant__)          v1 global (cudaMemcpy + acquire fence)
//   v2 global, qwords 8..15 zeroed        v3 param, qwords 8..15 zeroed
//   v4 global, published by tensormap.cp_fenceproxy from shared memory
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int V>
__global__ void k2(const __grid_constant__ CUtensorMap tm, CUtensorMap* gtm, double* out, int x0,
                   int y0) {
  __shared__ __align__(1024) double s[64];
  __shared__ __align__(128) CUtensorMap stm;
  __shared__ __align__(8) uint64_t bar;
  const void* desc = (V == 0 || V == 3) ? (const void*)&tm : (const void*)gtm;
  if (V == 4) {
    if (threadIdx.x < 16) reinterpret_cast<uint64_t*>(&stm)[threadIdx.x] = reinterpret_cast<const uint64_t*>(&tm)[threadIdx.x];
    __syncwarp();
    asm volatile(
        "tensormap.cp_fenceproxy.global.shared::cta.tensormap::generic.release.gpu.sync.aligned "
        "[%0], [%1], 128;" ::"l"(gtm),
        "r"(smem_u32(&stm))
        : "memory");
  }
  if (V == 1 || V == 2 || V == 4)
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(gtm) : "memory");
  if (V == 5) {  // converged issue: every thread reaches the copy, thread 0 predicated on
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" ::"r"(smem_u32(&bar)));
    }
    __syncthreads();
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.eq.u32 p, %5, 0;\n\t"
        "@p cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];\n\t}" ::"r"(smem_u32(s)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(smem_u32(&bar)), "r"(threadIdx.x)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW5:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W5;\n\t}" ::"r"(
            smem_u32(&bar)));
  } else if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" ::"r"(smem_u32(&bar)));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(s)),
        "l"(reinterpret_cast<uint64_t>(desc)), "r"(x0), "r"(y0), "r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  const int v = argc > 1 ? atoi(argv[1]) : 0;
  const int NX = 32, NY = 16;
  std::vector<double> h(NX * NY);
  for (int i = 0; i < NX * NY; ++i) h[i] = i;
  double *d, *o;
  CUtensorMap* gtm;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 64 * 8);
  cudaMalloc(&gtm, 128);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  memset(&tm, 0, sizeof tm);
  cuuint64_t dims[2] = {NX, NY};
  cuuint64_t strides[1] = {NX * 8ull};
  cuuint32_t box[2] = {8, 8};
  cuuint32_t es[2] = {1, 1};
  CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box,
                                      es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (v == 2 || v == 3)
    for (int i = 8; i < 16; ++i) reinterpret_cast<uint64_t*>(&tm)[i] = 0;
  cudaMemcpy(gtm, &tm, 128, cudaMemcpyHostToDevice);
  if (v == 0) k2<0><<<1, 32>>>(tm, gtm, o, 3, 2);
  if (v == 1) k2<1><<<1, 32>>>(tm, gtm, o, 3, 2);
  if (v == 2) k2<2><<<1, 32>>>(tm, gtm, o, 3, 2);
  if (v == 3) k2<3><<<1, 32>>>(tm, gtm, o, 3, 2);
  if (v == 4) k2<4><<<1, 32>>>(tm, gtm, o, 3, 2);
  if (v == 5) k2<5><<<1, 32>>>(tm, gtm, o, 3, 2);
  std::vector<double> s(64);
  cudaError_t e = cudaMemcpy(s.data(), o, 64 * 8, cudaMemcpyDeviceToHost);
  printf("v%d encode %d: %s; s[0]=%g (want %d) s[9]=%g (want %d)\n", v, (int)r, cudaGetErrorString(e),
         s[0], 2 * NX + 3, s[9], 3 * NX + 4);
  return 0;
}
