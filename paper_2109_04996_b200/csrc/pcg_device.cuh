// Device-side PCG helpers shared by the operator kernels and pcg_kernels.cu:
// the "last CTA" pattern that finalises a fixed-order reduction inside the
// kernel that produced the partials (no extra launch, no redundant work).
#pragma once
#include "hxf_device.cuh"
#include "hxf_internal.h"

namespace hxf {

// Returns true in every thread of the CTA that arrives last.  Thread 0 must
// have written this CTA's partial(s) before the call.
__device__ __forceinline__ bool pcg_last_cta(unsigned int* counter) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  return last;
}

// Fixed-order sum of n partials by the calling CTA (blockDim.x threads);
// result on thread 0.  L1-bypassing loads: the partials of other CTAs.
template <int NT>
__device__ __forceinline__ double pcg_sum_partials(const double* part, int n, double* scratch) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += NT) s += __ldcg(part + i);
  return block_sum<NT>(s, scratch);
}

// K1 epilogue: publish this CTA's p.(A p) partial; the last CTA sums all
// partials in a fixed order and adds the constrained rows' p.p (A p = p
// there): red[0] = this rank's pAp, all-reduced across ranks if partitioned.
template <int NT>
__device__ __forceinline__ void pcg_alpha_epilogue(const PcgAlphaFin& f, double* scratch) {
  if (!f.st) return;
  if (!pcg_last_cta(&f.st->counter[0])) return;
  // partials of earlier passes (f.nparts) followed by this launch's CTAs
  const double s = pcg_sum_partials<NT>(f.parts, f.nparts + (int)gridDim.x, scratch);
  if (threadIdx.x == 0) {
    f.st->counter[0] = 0;
    f.st->red[0] = s + f.st->red[3];
  }
}

}  // namespace hxf
