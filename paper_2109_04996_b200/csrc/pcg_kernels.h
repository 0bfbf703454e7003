// Device-resident PCG state and launchers (pcg_kernels.cu).
#pragma once
#include "hxf_internal.h"

namespace hxf {

enum PcgError { PCG_OK = 0, PCG_ERR_RHS = 1, PCG_ERR_APPLY_NAN = 2, PCG_ERR_INDEFINITE = 3,
                PCG_ERR_RESID = 4 };

struct PcgState {
  double rho[2];  // rho before iteration k lives in rho[k & 1]
  double pap, alpha, beta, norm_b, target, res, tol;
  int it, stop, converged, error, limit, fixed;
};

int vec_grid();
cudaError_t launch_init_y(cudaStream_t s, int64_t n_L, int m, const double* x, double* y,
                          const uint32_t* mask);
cudaError_t pcg_launch_init(cudaStream_t s, int64_t n_L, int m, const double* b, const double* d,
                            double* x, double* r, double* p, double* Ap, const uint32_t* mask,
                            double* part, PcgState* st, double* hist, double* cons_part);
cudaError_t pcg_launch_update(cudaStream_t s, PcgState* st, int it, const double* kpart, int gk,
                              const double* cpart, int gc, int64_t n, const double* d, double* x,
                              double* r, const double* p, const double* Ap, double* upart);
cudaError_t pcg_launch_direction(cudaStream_t s, PcgState* st, int it, const double* upart,
                                 double* hist, int64_t n_L, int m, const double* d,
                                 const double* r, double* p, double* Ap, const uint32_t* mask,
                                 double* cpart);

}  // namespace hxf
