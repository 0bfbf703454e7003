// TEST INFRASTRUCTURE ONLY — exercises the reference-side integration
// (integration/hexfem_hxf.cpp) on the UNMODIFIED reference's own objects:
// a hexfem::BpProblem built by the reference's bp_setup is applied / solved
// once by the reference (CPU) and once through hexfem::hxf_backend (the B200
// C-ABI), in the same process, so the GPU tests can compare the two.
#include <cstring>
#include <exception>
#include <memory>
#include <span>
#include <string>

#include "hexfem/bench.hpp"
#include "hexfem_hxf.hpp"

using namespace hexfem;

namespace {
thread_local std::string g_err;
struct H {
  BpProblem prob;
  std::unique_ptr<ThreadPool> pool;
};
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}
}  // namespace

extern "C" {

const char* orh_last_error() { return g_err.c_str(); }

void* orh_setup(int bp, int p, int nx, int ny, int nz, int deform, int threads) {
  H* out = nullptr;
  guarded([&] {
    auto h = std::make_unique<H>();
    h->pool = std::make_unique<ThreadPool>(threads);
    BpConfig c;
    c.bp = BpId(bp);
    c.p = p;
    c.dims = {nx, ny, nz};
    c.deformation = deform ? Deformation::Sine : Deformation::None;
    c.threads = threads;
    h->prob = bp_setup(c, h->pool.get());
    out = h.release();
  });
  return out;
}

void orh_free(void* h) { delete static_cast<H*>(h); }
int64_t orh_size(void* h) { return static_cast<H*>(h)->prob.op.size(); }

// which = 0: reference CPU operator_apply, 1: hexfem::hxf_backend::operator_apply
int orh_apply(void* hv, int which, const double* x, double* y) {
  auto* h = static_cast<H*>(hv);
  const size_t n = size_t(h->prob.op.size());
  return guarded([&] {
    if (which == 0)
      operator_apply(h->prob.op, {x, n}, {y, n}, h->pool.get());
    else
      hxf_backend::operator_apply(h->prob.op, {x, n}, {y, n});
  });
}

int orh_diagonal(void* hv, int which, double* d) {
  auto* h = static_cast<H*>(hv);
  return guarded([&] {
    auto v = which == 0 ? operator_diagonal(h->prob.op, h->pool.get())
                        : hxf_backend::operator_diagonal(h->prob.op);
    std::memcpy(d, v.data(), v.size() * sizeof(double));
  });
}

int orh_solve(void* hv, int which, double tol, int jacobi, double* x, int* iters, int* converged) {
  auto* h = static_cast<H*>(hv);
  return guarded([&] {
    h->prob.config.tol_rel = tol;
    h->prob.config.fixed_iterations = std::nullopt;
    auto res = which == 0 ? solve_bp(h->prob, h->pool.get(), jacobi != 0)
                          : hxf_backend::solve_bp(h->prob, nullptr, jacobi != 0);
    std::memcpy(x, res.x.data(), res.x.size() * sizeof(double));
    *iters = res.report.iterations;
    *converged = res.report.converged ? 1 : 0;
  });
}

void orh_release() { hxf_backend::release_all(); }

// Scale the operator's stored qdata in place (same addresses, new contents):
// the backend must notice and re-upload (its side table is content-checked).
void orh_scale_qdata(void* hv, double s) {
  auto& op = static_cast<H*>(hv)->prob.op;
  for (auto* qd : {&op.mass_qdata, &op.diff_qdata})
    if (qd->has_value())
      for (double& v : (*qd)->values) v *= s;
}

// operator_apply with a FlopCounter attached: which = 0 the reference's
// instrumented count, 1 the backend's credited count.
int orh_apply_counted(void* hv, int which, const double* x, double* y, uint64_t* flops) {
  auto* h = static_cast<H*>(hv);
  const size_t n = size_t(h->prob.op.size());
  return guarded([&] {
    FlopCounter fc;
    MatFreeOperator op = h->prob.op;  // a copy: same arrays (shared qdata), new address
    op.plan.flops = &fc;
    if (which == 0)
      operator_apply(op, {x, n}, {y, n}, h->pool.get());
    else
      hxf_backend::operator_apply(op, {x, n}, {y, n});
    *flops = fc.count();
  });
}

// Restriction surface on the problem's own ElemRestriction: what = 0 apply_g,
// 1 apply_g_transpose, 2 gather_scalar, 3 multiplicity.
int orh_restriction(void* hv, int which, int what, const double* in, int64_t n_in, double* out,
                    int64_t n_out) {
  auto* h = static_cast<H*>(hv);
  const auto& r = h->prob.op.restriction;
  return guarded([&] {
    std::span<const double> a(in, size_t(n_in));
    std::span<double> b(out, size_t(n_out));
    if (what == 0) which ? hxf_backend::apply_g(r, a, b) : apply_g(r, a, b, h->pool.get());
    if (what == 1)
      which ? hxf_backend::apply_g_transpose(r, a, b) : apply_g_transpose(r, a, b, h->pool.get());
    if (what == 2)
      which ? hxf_backend::gather_scalar(r, a, b) : gather_scalar(r, a, b, h->pool.get());
    if (what == 3) {
      auto m = which ? hxf_backend::multiplicity(r) : multiplicity(r);
      std::memcpy(out, m.data(), m.size() * sizeof(double));
    }
  });
}

// Basis surface on the problem's own TensorBasis: what = 0 apply_basis_batch
// (ne blocks), 1 apply_tensor_3d (m components); counted flops out.
int orh_basis(void* hv, int which, int what, int grad, int transpose, int64_t ne_or_m,
              const double* in, int64_t n_in, double* out, int64_t n_out, uint64_t* flops) {
  auto* h = static_cast<H*>(hv);
  const auto& basis = h->prob.basis;
  return guarded([&] {
    const EvalMode mode = grad ? EvalMode::Grad : EvalMode::Interp;
    const EvalDirection dir = transpose ? EvalDirection::Transpose : EvalDirection::Forward;
    std::span<const double> a(in, size_t(n_in));
    std::span<double> b(out, size_t(n_out));
    FlopCounter fc;
    KernelPlan plan;
    plan.p = basis.p;
    plan.q = basis.q;
    plan.flops = &fc;
    ContractionScratch scratch;
    if (what == 0)
      which ? hxf_backend::apply_basis_batch(plan, basis, mode, dir, ne_or_m, a, b, scratch)
            : apply_basis_batch(plan, basis, mode, dir, ne_or_m, a, b, scratch);
    else
      which ? hxf_backend::apply_tensor_3d(basis, mode, dir, int(ne_or_m), a, b)
            : apply_tensor_3d(basis, mode, dir, int(ne_or_m), a, b);
    *flops = fc.count();
  });
}

int orh_contract(int which, const double* M, int64_t m_len, int n_out, int n_in, int dim,
                 const int* shape, int64_t ne, const double* in, int64_t n_in_len, double* out,
                 int64_t n_out_len, int accumulate, uint64_t* flops) {
  return guarded([&] {
    FlopCounter fc;
    KernelPlan plan;
    plan.flops = &fc;
    std::span<const double> mm(M, size_t(m_len)), a(in, size_t(n_in_len));
    std::span<double> b(out, size_t(n_out_len));
    const std::array<int, 3> sh{shape[0], shape[1], shape[2]};
    if (which)
      hxf_backend::contract_batch(plan, mm, n_out, n_in, dim, sh, ne, a, b, accumulate != 0);
    else
      contract_batch(plan, mm, n_out, n_in, dim, sh, ne, a, b, accumulate != 0);
    *flops = fc.count();
  });
}

uint64_t orh_flops_estimate(int which, int p, int q, int m, int grad) {
  KernelPlan plan;
  plan.p = p;
  plan.q = q;
  plan.m = m;
  const EvalMode mode = grad ? EvalMode::Grad : EvalMode::Interp;
  return which ? hxf_backend::flops_estimate(plan, mode) : flops_estimate(plan, mode);
}

}  // extern "C"
