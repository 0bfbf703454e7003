// See hexfem_hxf.hpp.  MatFreeOperator / ElemRestriction are plain host
// structs with no slot for a device handle (operator.hpp:19-31,
// restriction.hpp:26-33), so the backend keeps a small side table of device
// copies.  An entry is found by the object's address, the identity and size
// of its arrays and its scalar parameters (p, q, m, E, n_L, alpha, beta), and
// is reused only while a sampled content fingerprint of those arrays still
// matches — a new object that lands on recycled addresses, or an in-place
// edit of qdata / indices / constraints, re-uploads instead of returning a
// stale operator.  The table is bounded (least recently used entries are
// dropped), and each entry serialises the host-staged calls made through it.
#include "hexfem_hxf.hpp"

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "hxf.h"

namespace hexfem::hxf_backend {
namespace {

void check(int status) {
  if (status == HXF_OK) return;
  const std::string msg = hxf_last_error();
  if (status == HXF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

constexpr size_t kMaxEntries = 8;

// FNV-1a over the size and up to 4096 evenly spaced 8-byte words (first and
// last included): O(1) per call, catches re-filled or re-sized arrays.
uint64_t fingerprint(const void* data, size_t bytes, uint64_t h = 1469598103934665603ull) {
  auto mix = [&h](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix(bytes);
  const size_t words = bytes / 8;
  if (!data || words == 0) return h;
  const auto* p = static_cast<const unsigned char*>(data);
  const size_t samples = std::min<size_t>(words, 4096);
  for (size_t i = 0; i < samples; ++i) {
    const size_t w = samples == 1 ? 0 : i * (words - 1) / (samples - 1);
    uint64_t v;
    std::memcpy(&v, p + 8 * w, 8);
    mix(v);
  }
  return h;
}

template <class T>
uint64_t fp_vec(const std::vector<T>& v, uint64_t h) {
  return fingerprint(v.data(), v.size() * sizeof(T), h);
}

uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

struct OpHandle {
  hxf_op* op = nullptr;
  std::mutex mu;  // host-staged calls share the handle's staging buffers
  ~OpHandle() {
    if (op) hxf_operator_destroy(op);
  }
};
struct RestrHandle {
  hxf_restr* r = nullptr;
  ~RestrHandle() {
    if (r) hxf_elem_restriction_destroy(r);
  }
};

template <class H>
struct Entry {
  std::vector<uint64_t> key;
  uint64_t fp = 0;
  uint64_t last_use = 0;
  std::shared_ptr<H> h;
};

std::mutex g_mu;          // the tables and the context
std::mutex g_scratch_mu;  // the context's staging buffers (restriction / basis / contraction)
hxf_ctx* g_ctx = nullptr;
uint64_t g_tick = 0;
std::vector<Entry<OpHandle>> g_ops;
std::vector<Entry<RestrHandle>> g_restrs;

hxf_ctx* ctx_locked() {
  if (!g_ctx) check(hxf_context_create(0, nullptr, &g_ctx));
  return g_ctx;
}

// Find (key, fp) in the table: a hit returns the cached handle; a key hit
// with a changed fingerprint drops the stale entry; a miss evicts the least
// recently used entry when full and builds a new one.
template <class H, class Make>
std::shared_ptr<H> lookup(std::vector<Entry<H>>& table, const std::vector<uint64_t>& key,
                          uint64_t fp, Make&& make) {
  std::lock_guard<std::mutex> lock(g_mu);
  ++g_tick;
  for (auto it = table.begin(); it != table.end(); ++it) {
    if (it->key != key) continue;
    if (it->fp == fp) {
      it->last_use = g_tick;
      return it->h;
    }
    table.erase(it);  // same address / sizes, different contents
    break;
  }
  if (table.size() >= kMaxEntries) {
    auto lru = std::min_element(table.begin(), table.end(),
                                [](const auto& a, const auto& b) { return a.last_use < b.last_use; });
    table.erase(lru);
  }
  auto h = std::make_shared<H>();
  make(ctx_locked(), *h);
  table.push_back(Entry<H>{key, fp, g_tick, h});
  return h;
}

std::vector<uint64_t> op_key(const MatFreeOperator& op) {
  return {uint64_t(uintptr_t(&op)),
          uint64_t(uintptr_t(op.restriction.indices.data())), op.restriction.indices.size(),
          uint64_t(uintptr_t(op.mass_qdata ? op.mass_qdata->values.data() : nullptr)),
          op.mass_qdata ? op.mass_qdata->values.size() : 0,
          uint64_t(uintptr_t(op.diff_qdata ? op.diff_qdata->values.data() : nullptr)),
          op.diff_qdata ? op.diff_qdata->values.size() : 0,
          uint64_t(uintptr_t(op.constrained.data())), op.constrained.size(),
          uint64_t(op.basis.p), uint64_t(op.basis.q), uint64_t(op.m),
          uint64_t(op.restriction.num_elements), uint64_t(op.restriction.n_L),
          bits(op.alpha), bits(op.beta)};
}

uint64_t op_fingerprint(const MatFreeOperator& op) {
  uint64_t h = fp_vec(op.restriction.indices, 1469598103934665603ull);
  if (op.mass_qdata) h = fp_vec(op.mass_qdata->values, h);
  if (op.diff_qdata) h = fp_vec(op.diff_qdata->values, h);
  h = fp_vec(op.constrained, h);
  h = fp_vec(op.basis.interp1d, h);
  return fp_vec(op.basis.grad1d, h);
}

std::shared_ptr<OpHandle> device_op(const MatFreeOperator& op) {
  return lookup(g_ops, op_key(op), op_fingerprint(op), [&](hxf_ctx* ctx, OpHandle& h) {
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
    check(hxf_operator_create(ctx, &d, &h.op));
  });
}

std::shared_ptr<RestrHandle> device_restr(const ElemRestriction& r) {
  const std::vector<uint64_t> key = {uint64_t(uintptr_t(&r)), uint64_t(uintptr_t(r.indices.data())),
                                     r.indices.size(), uint64_t(r.num_elements),
                                     uint64_t(r.elem_size), uint64_t(r.n_L), uint64_t(r.m)};
  return lookup(g_restrs, key, fp_vec(r.indices, 1469598103934665603ull),
                [&](hxf_ctx* ctx, RestrHandle& h) {
                  int p = 0;
                  while ((p + 1) * (p + 1) * (p + 1) < r.elem_size) ++p;
                  if ((p + 1) * (p + 1) * (p + 1) != r.elem_size || p < 1)
                    throw std::invalid_argument("make_restriction: elem_size is not (p+1)^3");
                  if (int64_t(r.indices.size()) != r.num_elements * r.elem_size)
                    throw std::invalid_argument("make_restriction: index table size mismatch");
                  const int dims[3] = {0, 0, 0};
                  check(hxf_elem_restriction_create(ctx, p, r.m, r.num_elements, r.n_L,
                                                    r.indices.data(), dims, &h.r));
                });
}

hxf_ctx* context() {
  std::lock_guard<std::mutex> lock(g_mu);
  return ctx_locked();
}

hxf_eval_mode mode_of(EvalMode m) { return m == EvalMode::Grad ? HXF_GRAD : HXF_INTERP; }
hxf_eval_dir dir_of(EvalDirection d) {
  return d == EvalDirection::Transpose ? HXF_TRANSPOSE : HXF_FORWARD;
}

void credit(FlopCounter* fc, uint64_t n) {
  if (fc && n) fc->ops.fetch_add(n, std::memory_order_relaxed);
}

}  // namespace

void operator_apply(const MatFreeOperator& op, std::span<const double> x, std::span<double> y,
                    ThreadPool*, OperatorScratch*) {
  const int64_t n = op.size();
  if (int64_t(x.size()) != n || int64_t(y.size()) != n)
    throw std::invalid_argument("operator_apply: shape mismatch");
  auto h = device_op(op);
  {
    std::lock_guard<std::mutex> lock(h->mu);
    check(hxf_operator_apply(h->op, x.data(), y.data(), HXF_HOST, nullptr));
  }
  // the reference counts B and B^T of every element, component and stage
  // (operator.cpp:92-138 through contract_batch): 2 chains x flops_estimate
  if (op.plan.flops) {
    const int64_t E = op.restriction.num_elements;
    uint64_t total = 0;
    if (op.alpha != 0.0) total += 2 * uint64_t(E) * hxf_flops_estimate(op.basis.p, op.basis.q, op.m, HXF_GRAD);
    if (op.beta != 0.0) total += 2 * uint64_t(E) * hxf_flops_estimate(op.basis.p, op.basis.q, op.m, HXF_INTERP);
    credit(op.plan.flops, total);
  }
}

std::vector<double> operator_diagonal(const MatFreeOperator& op, ThreadPool*) {
  std::vector<double> d(size_t(op.size()));
  auto h = device_op(op);
  std::lock_guard<std::mutex> lock(h->mu);
  check(hxf_operator_diagonal(h->op, d.data(), HXF_HOST));
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
  auto h = device_op(op);
  {
    std::lock_guard<std::mutex> lock(h->mu);
    check(hxf_pcg(h->op, b.data(), jacobi_diag.empty() ? nullptr : jacobi_diag.data(), &o, x.data(),
                  HXF_HOST, &rep));
  }
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

void apply_g(const ElemRestriction& r, std::span<const double> l_vec, std::span<double> e_vec,
             ThreadPool*) {
  auto h = device_restr(r);
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  check(hxf_elem_restriction_apply(h->r, 0, l_vec.data(), int64_t(l_vec.size()), e_vec.data(),
                                   int64_t(e_vec.size()), HXF_HOST));
}

void apply_g_transpose(const ElemRestriction& r, std::span<const double> e_vec,
                       std::span<double> l_vec, ThreadPool*) {
  auto h = device_restr(r);
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  check(hxf_elem_restriction_apply(h->r, 1, e_vec.data(), int64_t(e_vec.size()), l_vec.data(),
                                   int64_t(l_vec.size()), HXF_HOST));
}

std::vector<double> multiplicity(const ElemRestriction& r) {
  std::vector<double> out(size_t(r.n_L));
  auto h = device_restr(r);
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  check(hxf_elem_restriction_multiplicity(h->r, out.data(), int64_t(out.size()), HXF_HOST));
  return out;
}

void gather_scalar(const ElemRestriction& r, std::span<const double> e_scalar,
                   std::span<double> l_scalar, ThreadPool*) {
  auto h = device_restr(r);
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  check(hxf_elem_restriction_gather_scalar(h->r, e_scalar.data(), int64_t(e_scalar.size()),
                                           l_scalar.data(), int64_t(l_scalar.size()), HXF_HOST));
}

void contract_batch(const KernelPlan& plan, std::span<const double> matrix, int n_out, int n_in,
                    int dim, std::array<int, 3> in_shape, std::int64_t ne,
                    std::span<const double> in, std::span<double> out, bool accumulate) {
  uint64_t count = 0;
  hxf_ctx* ctx = context();
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  check(hxf_contract_batch(ctx, matrix.data(), int64_t(matrix.size()), n_out, n_in, dim,
                           in_shape.data(), ne, in.data(), int64_t(in.size()), out.data(),
                           int64_t(out.size()), accumulate ? 1 : 0, HXF_HOST, &count));
  credit(plan.flops, count);
}

void apply_basis_batch(const KernelPlan& plan, const TensorBasis& basis, EvalMode mode,
                       EvalDirection dir, std::int64_t ne, std::span<const double> in,
                       std::span<double> out, ContractionScratch&) {
  const int64_t nd = basis.num_nodes(), nq = basis.num_qpts();
  const bool grad = mode == EvalMode::Grad, fwd = dir == EvalDirection::Forward;
  const int64_t in_e = fwd ? nd : (grad ? 3 * nq : nq), out_e = fwd ? (grad ? 3 * nq : nq) : nd;
  if (int64_t(in.size()) < ne * in_e || int64_t(out.size()) < ne * out_e)
    throw std::invalid_argument("apply_basis_batch: buffer too small");
  hxf_ctx* ctx = context();
  {
    std::lock_guard<std::mutex> lock(g_scratch_mu);
    check(hxf_basis_apply(ctx, basis.p, basis.q, basis.interp1d.data(), basis.grad1d.data(),
                          mode_of(mode), dir_of(dir), ne, in.data(), out.data(), HXF_HOST));
  }
  // the instrumented count of ne single-component blocks (contraction.hpp:69-74)
  credit(plan.flops, uint64_t(ne) * hxf_flops_estimate(basis.p, basis.q, 1, mode_of(mode)));
}

std::uint64_t flops_estimate(const KernelPlan& plan, EvalMode mode) {
  return hxf_flops_estimate(plan.p, plan.q, plan.m, mode_of(mode));
}

void apply_tensor_3d(const TensorBasis& basis, EvalMode mode, EvalDirection dir, int m,
                     std::span<const double> u, std::span<double> v) {
  hxf_ctx* ctx = context();
  std::lock_guard<std::mutex> lock(g_scratch_mu);
  check(hxf_apply_tensor_3d(ctx, basis.p, basis.q, basis.interp1d.data(), basis.grad1d.data(),
                            mode_of(mode), dir_of(dir), m, u.data(), int64_t(u.size()), v.data(),
                            int64_t(v.size()), HXF_HOST));
}

void release(const MatFreeOperator& op) {
  std::lock_guard<std::mutex> lock(g_mu);
  const std::vector<uint64_t> key = op_key(op);
  g_ops.erase(std::remove_if(g_ops.begin(), g_ops.end(), [&](const auto& e) { return e.key == key; }),
              g_ops.end());
}

void release_all() {
  std::lock_guard<std::mutex> lock(g_mu);
  g_ops.clear();
  g_restrs.clear();
}

}  // namespace hexfem::hxf_backend
