// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A flat C interface over the UNMODIFIED reference library (hexfem, built
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It
// exposes exactly the same `orc_*` entry points as the C restatement in
// oracle/hexfem_oracle.c, so a test can swap "the reference itself" for "our
// restatement of it" and compare them value for value.
//
// Every function forwards to the reference's own public API:
//   orc_setup      -> hexfem::bp_setup            (proj/src/bench.cpp:64-119)
//   orc_apply      -> hexfem::operator_apply      (proj/src/operator.cpp:64-144)
//   orc_diagonal   -> hexfem::operator_diagonal   (proj/src/operator.cpp:170-256)
//   orc_solve      -> hexfem::solve_bp / pcg      (proj/src/bench.cpp:121-137)
//   orc_l2_error   -> hexfem::l2_error            (proj/src/bench.cpp:139-189)
//   orc_quadrature -> hexfem::make_quadrature     (proj/src/quadrature.cpp:66-126)
//   orc_basis      -> hexfem::make_basis          (proj/src/tensor_basis.cpp:40-71)
//   orc_apply_basis-> hexfem::apply_basis_batch   (proj/src/contraction.cpp:248-332)
//   orc_run_bench  -> hexfem::run_bench           (proj/src/bench.cpp:191-229)
//   orc_sweep_model-> hexfem::run_scaling_sweep + sweep_csv with the synthetic
//                     timing model of tests/test_bench.cpp:142-150
//   orc_record_json-> hexfem::bench_record_json   (proj/src/bench.cpp:351-363)
#include <array>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "hexfem/bench.hpp"

using namespace hexfem;

namespace {
thread_local std::string g_err;

struct RefProblem {
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

const char* orc_last_error() { return g_err.c_str(); }
const char* orc_impl_name() { return "reference"; }

void* orc_setup(int bp, int p, int nx, int ny, int nz, int deform, int threads) {
  RefProblem* out = nullptr;
  int rc = guarded([&] {
    auto rp = std::make_unique<RefProblem>();
    rp->pool = std::make_unique<ThreadPool>(threads < 1 ? 1 : threads);
    BpConfig c;
    c.bp = BpId(bp);
    c.p = p;
    c.dims = {nx, ny, nz};
    c.deformation = deform ? Deformation::Sine : Deformation::None;
    c.threads = threads < 1 ? 1 : threads;
    rp->prob = bp_setup(c, rp->pool.get());
    out = rp.release();
  });
  return rc == 0 ? out : nullptr;
}

void orc_free(void* h) { delete static_cast<RefProblem*>(h); }

// info[0..9] = m, n_L, E, S, nq, q, n_dofs, n_constrained, p, nodes_per_axis_x
void orc_info(void* h, int64_t* info) {
  auto* rp = static_cast<RefProblem*>(h);
  const auto& pr = rp->prob;
  info[0] = pr.m;
  info[1] = pr.mesh.n_L;
  info[2] = pr.mesh.num_elements();
  info[3] = pr.mesh.nodes_per_elem();
  info[4] = pr.basis.num_qpts();
  info[5] = pr.basis.q;
  info[6] = pr.n_dofs;
  info[7] = int64_t(pr.op.constrained.size());
  info[8] = pr.basis.p;
  info[9] = pr.mesh.nodes_per_axis[0];
}

const double* orc_rhs(void* h) { return static_cast<RefProblem*>(h)->prob.rhs.data(); }
const double* orc_exact(void* h) {
  return static_cast<RefProblem*>(h)->prob.exact_nodal.data();
}
const double* orc_coords(void* h) {
  return static_cast<RefProblem*>(h)->prob.mesh.coords.data();
}
const int64_t* orc_indices(void* h) {
  return static_cast<RefProblem*>(h)->prob.op.restriction.indices.data();
}
const int64_t* orc_constrained(void* h) {
  return static_cast<RefProblem*>(h)->prob.op.constrained.data();
}
// kind 0 = mass, 1 = diffusion.  bp_setup keeps only the qdata the operator
// uses (bench.cpp:113-115), so the other one is NULL.
const double* orc_qdata(void* h, int kind) {
  const auto& op = static_cast<RefProblem*>(h)->prob.op;
  if (kind == 0) return op.mass_qdata ? op.mass_qdata->values.data() : nullptr;
  return op.diff_qdata ? op.diff_qdata->values.data() : nullptr;
}
const double* orc_interp1d(void* h) {
  return static_cast<RefProblem*>(h)->prob.basis.interp1d.data();
}
const double* orc_grad1d(void* h) {
  return static_cast<RefProblem*>(h)->prob.basis.grad1d.data();
}
double orc_alpha(void* h) { return static_cast<RefProblem*>(h)->prob.op.alpha; }
double orc_beta(void* h) { return static_cast<RefProblem*>(h)->prob.op.beta; }

int orc_apply(void* h, const double* x, double* y) {
  auto* rp = static_cast<RefProblem*>(h);
  const std::size_t n = std::size_t(rp->prob.op.size());
  return guarded([&] {
    operator_apply(rp->prob.op, std::span<const double>(x, n), std::span<double>(y, n),
                   rp->pool.get());
  });
}

int orc_diagonal(void* h, double* d) {
  auto* rp = static_cast<RefProblem*>(h);
  return guarded([&] {
    auto v = operator_diagonal(rp->prob.op, rp->pool.get());
    std::memcpy(d, v.data(), v.size() * sizeof(double));
  });
}

// fixed_iters < 0: solve mode.  hist receives up to hist_cap residual norms.
int orc_solve(void* h, double tol, int max_iter, int jacobi, int fixed_iters, double* x,
              double* hist, int hist_cap, int* iters, int* converged) {
  auto* rp = static_cast<RefProblem*>(h);
  return guarded([&] {
    rp->prob.config.tol_rel = tol;
    rp->prob.config.max_iter = max_iter;
    rp->prob.config.fixed_iterations =
        fixed_iters >= 0 ? std::optional<int>(fixed_iters) : std::nullopt;
    auto res = solve_bp(rp->prob, rp->pool.get(), jacobi != 0);
    std::memcpy(x, res.x.data(), res.x.size() * sizeof(double));
    const int nh = int(res.report.residual_history.size());
    for (int i = 0; i < nh && i < hist_cap; ++i) hist[i] = res.report.residual_history[i];
    *iters = res.report.iterations;
    *converged = res.report.converged ? 1 : 0;
  });
}

double orc_l2_error(void* h, const double* u) {
  auto* rp = static_cast<RefProblem*>(h);
  const std::size_t n = std::size_t(rp->prob.op.size());
  return l2_error(rp->prob.mesh, rp->prob.m, std::span<const double>(u, n),
                  manufactured_solution);
}

// kind 0 = Gauss-Legendre, 1 = Gauss-Lobatto-Legendre
int orc_quadrature(int kind, int q, double* pts, double* wts) {
  return guarded([&] {
    auto r = make_quadrature(kind ? QuadratureKind::GaussLobattoLegendre
                                  : QuadratureKind::GaussLegendre, q);
    std::memcpy(pts, r.points.data(), sizeof(double) * q);
    std::memcpy(wts, r.weights.data(), sizeof(double) * q);
  });
}

int orc_basis(int p, int kind, int q, double* interp, double* grad) {
  return guarded([&] {
    auto b = make_basis(p, make_quadrature(kind ? QuadratureKind::GaussLobattoLegendre
                                                : QuadratureKind::GaussLegendre, q));
    std::memcpy(interp, b.interp1d.data(), sizeof(double) * b.interp1d.size());
    std::memcpy(grad, b.grad1d.data(), sizeof(double) * b.grad1d.size());
  });
}

// mode 0 interp / 1 grad; dir 0 forward / 1 transpose
int orc_apply_basis(int p, int kind, int q, int mode, int dir, int64_t ne, const double* in,
                    int64_t n_in, double* out, int64_t n_out) {
  return guarded([&] {
    auto b = make_basis(p, make_quadrature(kind ? QuadratureKind::GaussLobattoLegendre
                                                : QuadratureKind::GaussLegendre, q));
    KernelPlan plan;
    plan.p = p;
    plan.q = q;
    ContractionScratch scratch;
    apply_basis_batch(plan, b, mode ? EvalMode::Grad : EvalMode::Interp,
                      dir ? EvalDirection::Transpose : EvalDirection::Forward, ne,
                      std::span<const double>(in, std::size_t(n_in)),
                      std::span<double>(out, std::size_t(n_out)), scratch);
  });
}

int orc_contract_batch(const double* M, int64_t m_len, int n_out, int n_in, int dim,
                       const int* shape, int64_t ne, const double* in, int64_t in_len, double* out,
                       int64_t out_len, int accumulate, uint64_t* flops) {
  return guarded([&] {
    FlopCounter counter;
    KernelPlan plan;
    plan.flops = flops ? &counter : nullptr;
    contract_batch(plan, std::span<const double>(M, std::size_t(m_len)), n_out, n_in, dim,
                   std::array<int, 3>{shape[0], shape[1], shape[2]}, ne,
                   std::span<const double>(in, std::size_t(in_len)),
                   std::span<double>(out, std::size_t(out_len)), accumulate != 0);
    if (flops) *flops += counter.count();
  });
}

int orc_apply_tensor_3d(int p, int kind, int q, int mode, int dir, int m, const double* u,
                        int64_t u_len, double* v, int64_t v_len) {
  return guarded([&] {
    auto b = make_basis(p, make_quadrature(kind ? QuadratureKind::GaussLobattoLegendre
                                                : QuadratureKind::GaussLegendre, q));
    apply_tensor_3d(b, mode ? EvalMode::Grad : EvalMode::Interp,
                    dir ? EvalDirection::Transpose : EvalDirection::Forward, m,
                    std::span<const double>(u, std::size_t(u_len)),
                    std::span<double>(v, std::size_t(v_len)));
  });
}

uint64_t orc_flops_estimate(int p, int q, int m, int mode) {
  KernelPlan plan;
  plan.p = p;
  plan.q = q;
  plan.m = m;
  return flops_estimate(plan, mode ? EvalMode::Grad : EvalMode::Interp);
}

int orc_apply_basis_counted(int p, int kind, int q, int mode, int dir, int64_t ne,
                            const double* in, int64_t n_in, double* out, int64_t n_out,
                            uint64_t* flops) {
  return guarded([&] {
    auto b = make_basis(p, make_quadrature(kind ? QuadratureKind::GaussLobattoLegendre
                                                : QuadratureKind::GaussLegendre, q));
    FlopCounter counter;
    KernelPlan plan;
    plan.p = p;
    plan.q = q;
    plan.flops = &counter;
    ContractionScratch scratch;
    apply_basis_batch(plan, b, mode ? EvalMode::Grad : EvalMode::Interp,
                      dir ? EvalDirection::Transpose : EvalDirection::Forward, ne,
                      std::span<const double>(in, std::size_t(n_in)),
                      std::span<double>(out, std::size_t(n_out)), scratch);
    if (flops) *flops += counter.count();
  });
}

int orc_gather_scalar(void* h, const double* e_scalar, int64_t e_len, double* l_scalar,
                      int64_t l_len) {
  return guarded([&] {
    gather_scalar(static_cast<RefProblem*>(h)->prob.op.restriction,
                  std::span<const double>(e_scalar, std::size_t(e_len)),
                  std::span<double>(l_scalar, std::size_t(l_len)));
  });
}

// The reference benchmark record (bench.cpp:191-229): returns dofs_rate and
// fills rec[] = {n, iterations, seconds, E, q}.
int orc_run_bench(int bp, int p, int nx, int ny, int nz, int deform, int threads, int iters,
                  double* rec) {
  return guarded([&] {
    BpConfig c;
    c.bp = BpId(bp);
    c.p = p;
    c.dims = {nx, ny, nz};
    c.deformation = deform ? Deformation::Sine : Deformation::None;
    c.threads = threads;
    c.fixed_iterations = iters;
    auto r = run_bench(c);
    rec[0] = double(r.n);
    rec[1] = r.iterations;
    rec[2] = r.seconds;
    rec[3] = double(r.E);
    rec[4] = r.q;
    rec[5] = r.dofs_rate;
  });
}

// Scaling sweep under the timing model T(n,1) = a n, T(n,P>1) = a n / P + b
// (the reference's own test model): writes sweep_csv() into csv (NUL-terminated,
// cap bytes) and summary = {r_max, n08 (or -1), work_constant}.
int orc_sweep_model(int bp, int p, const int* dims, int ndims, const int* threads, int nthreads,
                    int iters, double a, double b, char* csv, int64_t cap, double* summary) {
  return guarded([&] {
    std::vector<std::array<int, 3>> dl;
    for (int i = 0; i < ndims; ++i) dl.push_back({dims[3 * i], dims[3 * i + 1], dims[3 * i + 2]});
    std::vector<int> tl(threads, threads + nthreads);
    const TimingModel model = [&](std::int64_t n, int P) {
      return P == 1 ? a * double(n) : a * double(n) / P + b;
    };
    const auto res = run_scaling_sweep(BpId(bp), p, dl, tl, iters, Deformation::None, model);
    const std::string text = sweep_csv(res);
    if (int64_t(text.size()) + 1 > cap) throw std::invalid_argument("orc_sweep_model: buffer");
    std::memcpy(csv, text.c_str(), text.size() + 1);
    summary[0] = res.summary.r_max;
    summary[1] = res.summary.n08_per_rank ? *res.summary.n08_per_rank : -1.0;
    summary[2] = res.summary.work_constant;
  });
}

int orc_record_json(const char* bp, int p, int q, int64_t E, int64_t n, int P, int iters,
                    double seconds, double dofs_rate, double n_per_rank, char* out, int64_t cap) {
  return guarded([&] {
    BenchRecord r;
    r.bp = bp;
    r.p = p;
    r.q = q;
    r.E = E;
    r.n = n;
    r.P = P;
    r.iterations = iters;
    r.seconds = seconds;
    r.dofs_rate = dofs_rate;
    r.n_per_rank = n_per_rank;
    const std::string text = bench_record_json(r);
    if (int64_t(text.size()) + 1 > cap) throw std::invalid_argument("orc_record_json: buffer");
    std::memcpy(out, text.c_str(), text.size() + 1);
  });
}

}  // extern "C"
