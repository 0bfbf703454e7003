#include <cuda.h>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
extern "C" __global__ void k2(const __grid_constant__ CUtensorMap tm, double* out, int x0, int y0, int dst_off) {
  __shared__ __align__(1024) double sbuf[256];
  double* s = sbuf + dst_off;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 768;" ::"r"(smem_u32(&bar)));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(s)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(y0), "r"(smem_u32(&bar))
        : "memory");
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 64; i += blockDim.x) out[i] = s[i];
}
