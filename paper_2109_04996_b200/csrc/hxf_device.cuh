// Device-side primitives shared by every hxf kernel (sm_100a only).
//
// Bulk async copy (TMA engine, cp.async.bulk) + mbarrier transaction counts
// stream the per-element geometric factors into shared memory; FP64 RED
// (red.global.add.f64, SASS REDG.E.ADD.F64) performs the element-to-node
// scatter-add G^T without read-back.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "hxf kernels target sm_100a (B200) only"
#endif

namespace hxf {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n"
      "DONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// One bulk copy global -> shared (bytes % 16 == 0, both addresses 16B
// aligned), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Bulk prefetch of a global range into L2 (bytes % 16 == 0, 16B aligned).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Generic-proxy smem writes must be ordered before a later async-proxy (bulk
// copy) write into the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Programmatic dependent launch (launch attribute set by launch_pdl): wait
// until the preceding kernel in the stream has completed and its writes are
// visible (a no-op when launched without the attribute); let the next kernel
// launch early (it waits in its own pdl_wait, so this is safe anywhere).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

__device__ __forceinline__ void red_add(double* p, double v) {
  asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// predicated RED (no branch / reconvergence around the atomic)
__device__ __forceinline__ void red_add_if(double* p, double v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
      "d"(v), "r"((int)pred)
      : "memory");
}

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Division by a run-time invariant d (1 <= d < 2^31) for numerators n < 2^31
// with one IMAD.HI + shift (round-up magic number, as in CUTLASS FastDivmod),
// instead of the ~20-instruction integer division sequence.
struct FastDiv {
  uint32_t d, mul, shr;
  __device__ __forceinline__ explicit FastDiv(uint32_t den) : d(den), mul(0), shr(0) {
    if (den > 1) {
      const uint32_t l = 32 - __clz(den - 1);  // ceil(log2 den)
      const uint32_t p = 31 + l;
      mul = (uint32_t)(((1ull << p) + den - 1) / den);
      shr = p - 32;
    }
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return mul ? (__umulhi(n, mul) >> shr) : n;
  }
};

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block reduction (deterministic for a fixed block size).
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch /* >= NT/32 */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < (NT + 31) / 32; ++i) r += scratch[i];
  }
  __syncthreads();
  return r;  // valid on thread 0
}

}  // namespace hxf
