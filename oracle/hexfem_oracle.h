/* TEST INFRASTRUCTURE ONLY — the CPU oracle.  Never linked into, loaded by or
 * called from the product path (paper_2109_04996_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may use it, and only as the checker.
 *
 * A plain-C restatement of the reference (hexfem) algorithm for the BP1-BP6
 * operator-apply + Jacobi-PCG path, following the reference's operation order
 * (and compiled, like it, with -ffp-contract=off) so that it reproduces the
 * reference bit for bit; tests/test_oracle_ref.py checks exactly that against
 * the reference built from its own sources (oracle/_ref), and
 * tests/test_oracle_golden.py against the committed golden vectors and the
 * reference's own known-answer tests.
 *
 * The entry points mirror oracle/ref_shim/ref_capi.cpp one for one. */
#ifndef HEXFEM_ORACLE_H
#define HEXFEM_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
const char* orc_impl_name(void);

void* orc_setup(int bp, int p, int nx, int ny, int nz, int deform, int threads);
void orc_free(void* h);
void orc_info(void* h, int64_t* info);
const double* orc_rhs(void* h);
const double* orc_exact(void* h);
const double* orc_coords(void* h);
const int64_t* orc_indices(void* h);
const int64_t* orc_constrained(void* h);
const double* orc_qdata(void* h, int kind);
const double* orc_interp1d(void* h);
const double* orc_grad1d(void* h);
double orc_alpha(void* h);
double orc_beta(void* h);
int orc_apply(void* h, const double* x, double* y);
int orc_diagonal(void* h, double* d);
int orc_solve(void* h, double tol, int max_iter, int jacobi, int fixed_iters, double* x,
              double* hist, int hist_cap, int* iters, int* converged);
double orc_l2_error(void* h, const double* u);
int orc_quadrature(int kind, int q, double* pts, double* wts);
int orc_basis(int p, int kind, int q, double* interp, double* grad);
int orc_apply_basis(int p, int kind, int q, int mode, int dir, int64_t ne, const double* in,
                    int64_t n_in, double* out, int64_t n_out);

#ifdef __cplusplus
}
#endif
#endif
