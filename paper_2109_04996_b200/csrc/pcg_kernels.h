// Device-resident PCG launchers (pcg_kernels.cu).  d / dinv conventions:
// the init kernel takes the Jacobi diagonal d (or nullptr) and writes
// dinv = 1/d, which the update and direction kernels take as their `d`.
// own: owner bitmask over scalar nodes (partitioned problems), nullptr = all.
#pragma once
#include "hxf_internal.h"

namespace hxf {

int vec_grid();
cudaError_t launch_init_y(cudaStream_t s, int64_t n_L, int m, const double* x, double* y,
                          const uint32_t* mask, const uint32_t* own = nullptr);
cudaError_t pcg_launch_init(cudaStream_t s, PcgState* st, int64_t n_L, int m, const double* b,
                            const double* d, double* dinv, double* x, double* r, double* p,
                            double* Ap, const uint32_t* mask, const uint32_t* own, double* part);
cudaError_t pcg_launch_init_finalize(cudaStream_t s, PcgState* st, double* hist);
cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int it, int64_t n_L, int m,
                              const double* d, double* r, const double* Ap, const uint32_t* own,
                              double* part, int rev = 0);
// xmode 0: x += alpha p; 1: x update deferred (p_next -> pout, p kept); 2:
// x += alpha_prev pprev + alpha p (x updates of iteration pairs batched: one
// vector pass less per two iterations)
cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int it, double* hist, int64_t n_L,
                                 int m, const double* d, const double* r, double* x, const double* p,
                                 const double* pprev, double* pout, double* Ap,
                                 const uint32_t* mask, const uint32_t* own, double* part,
                                 int rev, int xmode);

// Fused update + direction (single domain, no owner mask, 16-byte aligned
// vectors, even n_L): one persistent cooperative kernel per iteration, a grid
// barrier between the two phases; the z = r/d of each CTA's chunk stays in
// shared memory across it.  ap_zero: Ap is zeroed in phase 1 right after it is
// read (the next operator kernel stores Ap = p on the constrained rows itself)
// and phase 2 writes no Ap preset.
bool pcg_step_fusable(int64_t n_L, const double* d, const double* r, double* x, const double* p,
                      const double* pprev, double* pout, double* Ap);
cudaError_t pcg_launch_step(cudaStream_t s, PcgState* st, int it, double* hist, int64_t n_L, int m,
                            const double* d, double* r, double* x, const double* p,
                            const double* pprev, double* pout, double* Ap, const uint32_t* mask,
                            double* part, int rev, int xmode, bool ap_zero = false);
int pcg_step_grid();  // CTAs of the fused kernel (partials it writes: 3 per CTA)
void pcg_step_timestamps(int on, unsigned long long* out);  // measurement only

}  // namespace hxf
