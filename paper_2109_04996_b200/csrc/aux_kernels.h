// Launchers for the API-surface / setup kernels (aux_kernels.cu).
#pragma once
#include "hxf_internal.h"

namespace hxf {

// Structured-box lattice description shared by the setup kernels.
struct Lattice {
  int p, S;           // degree, (p+1)^3
  int64_t E, n_L;     // elements, scalar nodes
  int64_t NX, NY;     // nodes per axis (x, y)
  int nx, ny, nz;     // elements per axis
};

cudaError_t launch_basis_apply(cudaStream_t s, int p, int q, const double* B, const double* G,
                               const double* Bt, const double* Gt, int mode, int dir, int64_t ne,
                               const double* in, double* out);
// structured-box setup fields: axes = [cx | cy | cz | sx | sy | sz] (global
// node counts gdim), the local box of ldim nodes at node offset off
cudaError_t launch_box_fields(cudaStream_t s, const double* axes, const int64_t gdim[3],
                              const int64_t off[3], const int64_t ldim[3], int deform, int m,
                              int poisson, double* coords, double* f, double* u);
// contract_batch: one 1-D contraction of ne element blocks (device M, n_out x n_in)
cudaError_t launch_contract_batch(cudaStream_t s, const double* M, int n_out, int n_in, int dim,
                                  const int shape[3], int64_t ne, const double* in, double* out,
                                  bool accumulate);
cudaError_t launch_qfunction(cudaStream_t s, int kind, const double* qd, int nq, int64_t e0,
                             int64_t ne, const double* u, double* v);
cudaError_t launch_restriction(cudaStream_t s, const Lattice& L, const int* idx, bool colorable,
                               int m, bool transpose, const double* in, double* out);
cudaError_t launch_multiplicity(cudaStream_t s, const Lattice& L, const int* idx, double* mult);
cudaError_t launch_qdata(cudaStream_t s, const Lattice& L, const int* idx, int q,
                         const double* B, const double* G, const double* w1,
                         const double* coords, int kind, double* vals, double* scratch,
                         int64_t batch, unsigned long long* fail_key, double* fail_det);
cudaError_t launch_diagonal(cudaStream_t s, const Lattice& L, const int* idx, bool colorable, int q,
                            const double* bb, const double* dd, const double* bd,
                            const double* mass_qd, int64_t mass_stride, const double* diff_qd,
                            int64_t diff_stride, double alpha, double beta, int m,
                            const uint32_t* cons_mask, double* ediag, double* ldiag, double* d);

}  // namespace hxf
