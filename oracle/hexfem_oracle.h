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
/* contract_batch (src/contraction.cpp:177-206) with the FlopCounter
 * (*flops += 2 per multiply-add, when flops != NULL). */
int orc_contract_batch(const double* M, int64_t m_len, int n_out, int n_in, int dim,
                       const int* shape, int64_t ne, const double* in, int64_t in_len, double* out,
                       int64_t out_len, int accumulate, uint64_t* flops);
/* apply_tensor_3d (src/tensor_basis.cpp:73-99) */
int orc_apply_tensor_3d(int p, int kind, int q, int mode, int dir, int m, const double* u,
                        int64_t u_len, double* v, int64_t v_len);
/* flops_estimate (src/contraction.cpp:334-340) */
uint64_t orc_flops_estimate(int p, int q, int m, int mode);
/* apply_basis_batch with a FlopCounter attached: the instrumented count */
int orc_apply_basis_counted(int p, int kind, int q, int mode, int dir, int64_t ne,
                            const double* in, int64_t n_in, double* out, int64_t n_out,
                            uint64_t* flops);
/* gather_scalar (src/restriction.cpp:86-106) over the problem's restriction */
int orc_gather_scalar(void* h, const double* e_scalar, int64_t e_len, double* l_scalar,
                      int64_t l_len);

#ifdef __cplusplus
}
#endif
#endif
