// See hexfem_hxf.hpp.  MatFreeOperator is a plain host struct with no slot for
// a device handle (operator.hpp:19-31), so the backend keeps a side table
// keyed on the operator's address and the identity of its arrays (indices,
// qdata, constraint list); a changed key re-uploads.
#include "hexfem_hxf.hpp"

#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "hxf.h"

namespace hexfem::hxf_backend {
namespace {

void check(int status) {
  if (status == HXF_OK) return;
  const std::string msg = hxf_last_error();
  if (status == HXF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

using Key = std::tuple<const void*, const void*, const void*, const void*, const void*, size_t>;

struct Entry {
  hxf_op* op = nullptr;
};

std::mutex g_mu;
hxf_ctx* g_ctx = nullptr;
std::map<Key, Entry> g_ops;

Key key_of(const MatFreeOperator& op) {
  return Key{&op, op.restriction.indices.data(),
             op.mass_qdata ? op.mass_qdata->values.data() : nullptr,
             op.diff_qdata ? op.diff_qdata->values.data() : nullptr, op.constrained.data(),
             op.constrained.size()};
}

hxf_op* device_op(const MatFreeOperator& op) {
  std::lock_guard<std::mutex> lock(g_mu);
  if (!g_ctx) check(hxf_context_create(0, nullptr, &g_ctx));
  const Key k = key_of(op);
  auto it = g_ops.find(k);
  if (it != g_ops.end()) return it->second.op;
  hxf_operator_desc d{};
  d.p = op.basis.p;
  d.q = op.basis.q;
  d.m = op.m;
  d.num_elements = op.restriction.num_elements;
  d.n_L = op.restriction.n_L;
  d.interp1d = op.basis.interp1d.data();
  d.grad1d = op.basis.grad1d.data();
  d.qpoints = op.basis.quad.points.data();
  d.indices = op.restriction.indices.data();  // verified bit-exact against the box lattice
  d.mass_qdata = op.mass_qdata ? op.mass_qdata->values.data() : nullptr;
  d.diff_qdata = op.diff_qdata ? op.diff_qdata->values.data() : nullptr;
  d.qdata_space = HXF_HOST;
  d.alpha = op.alpha;
  d.beta = op.beta;
  d.constrained = op.constrained.data();
  d.n_constrained = int64_t(op.constrained.size());
  d.block = op.plan.block;
  hxf_op* h = nullptr;
  check(hxf_operator_create(g_ctx, &d, &h));
  g_ops[k] = Entry{h};
  return h;
}

}  // namespace

void operator_apply(const MatFreeOperator& op, std::span<const double> x, std::span<double> y,
                    ThreadPool*, OperatorScratch*) {
  const int64_t n = op.size();
  if (int64_t(x.size()) != n || int64_t(y.size()) != n)
    throw std::invalid_argument("operator_apply: shape mismatch");
  check(hxf_operator_apply(device_op(op), x.data(), y.data(), HXF_HOST, nullptr));
}

std::vector<double> operator_diagonal(const MatFreeOperator& op, ThreadPool*) {
  std::vector<double> d(size_t(op.size()));
  check(hxf_operator_diagonal(device_op(op), d.data(), HXF_HOST));
  return d;
}

SolveReport pcg(const MatFreeOperator& op, std::span<const double> b,
                std::span<const double> jacobi_diag, const PcgOptions& options,
                std::span<double> x) {
  const int64_t n = op.size();
  if (int64_t(b.size()) != n || int64_t(x.size()) != n)
    throw std::invalid_argument("pcg: vector length mismatch");
  if (!jacobi_diag.empty() && int64_t(jacobi_diag.size()) != n)
    throw std::invalid_argument("pcg: preconditioner length mismatch");
  hxf_pcg_options o{};
  o.time_apply = 1;  // SolveReport::apply_time_seconds as the reference fills it
  o.tol_rel = options.tol_rel;
  o.max_iter = options.max_iter;
  o.fixed_iterations = options.fixed_iterations ? *options.fixed_iterations : -1;
  const int cap = (options.fixed_iterations ? *options.fixed_iterations : options.max_iter) + 2;
  std::vector<double> hist(static_cast<size_t>(cap));
  hxf_solve_report rep{};
  rep.residual_history = hist.data();
  rep.history_capacity = cap;
  check(hxf_pcg(device_op(op), b.data(), jacobi_diag.empty() ? nullptr : jacobi_diag.data(), &o,
                x.data(), HXF_HOST, &rep));
  SolveReport out;
  out.iterations = rep.iterations;
  out.converged = rep.converged != 0;
  out.residual_history.assign(hist.begin(), hist.begin() + rep.iterations + 1);
  out.apply_time_seconds = rep.apply_time_seconds;
  out.total_time_seconds = rep.total_time_seconds;
  return out;
}

BpSolveResult solve_bp(const BpProblem& problem, ThreadPool*, bool jacobi) {
  BpSolveResult result;
  result.x.assign(problem.rhs.size(), 0.0);
  std::vector<double> diag;
  if (jacobi) diag = hxf_backend::operator_diagonal(problem.op);
  PcgOptions opts;
  opts.tol_rel = problem.config.tol_rel;
  opts.max_iter = problem.config.max_iter;
  opts.fixed_iterations = problem.config.fixed_iterations;
  result.report = hxf_backend::pcg(problem.op, problem.rhs, diag, opts, result.x);
  return result;
}

void release_all() {
  std::lock_guard<std::mutex> lock(g_mu);
  for (auto& kv : g_ops) hxf_operator_destroy(kv.second.op);
  g_ops.clear();
}

}  // namespace hexfem::hxf_backend
