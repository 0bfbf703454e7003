// TEST INFRASTRUCTURE ONLY — exercises the reference-side integration
// (integration/hexfem_hxf.cpp) on the UNMODIFIED reference's own objects:
// a hexfem::BpProblem built by the reference's bp_setup is applied / solved
// once by the reference (CPU) and once through hexfem::hxf_backend (the B200
// C-ABI), in the same process, so the GPU tests can compare the two.
#include <cstring>
#include <exception>
#include <memory>
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

}  // extern "C"
