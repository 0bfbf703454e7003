// Device-resident PCG state and launchers (pcg_kernels.cu).
#pragma once
#include "hxf_internal.h"

namespace hxf {

int vec_grid();
cudaError_t launch_init_y(cudaStream_t s, int64_t n_L, int m, const double* x, double* y,
                          const uint32_t* mask);
// d: Jacobi diagonal or nullptr; dinv receives 1/d, the operand the update
// and direction kernels take as `d` (z = r * dinv).
cudaError_t pcg_launch_init(cudaStream_t s, PcgState* st, int64_t n_L, int m, const double* b,
                            const double* d, double* dinv, double* x, double* r, double* p,
                            double* Ap, const uint32_t* mask, double* part, double* hist);
cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int it, int64_t n, const double* d,
                              double* x, double* r, const double* p, const double* Ap,
                              double* part, double* hist);
cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int64_t n_L, int m,
                                 const double* d, const double* r, double* p, double* Ap,
                                 const uint32_t* mask, double* part);

}  // namespace hxf
