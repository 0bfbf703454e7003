// The reference's restriction / contraction / tensor-basis API surface in the
// host mirror (restriction.hpp:14-50, contraction.hpp:13-75,
// tensor_basis.hpp:35-47), over the C-ABI of include/hxf.h.
#include <mutex>

#include "hexfem_b200.hpp"

namespace hexfem_b200 {

namespace {
hxf_eval_mode mode_of(EvalMode m) { return m == EvalMode::Grad ? HXF_GRAD : HXF_INTERP; }
hxf_eval_dir dir_of(EvalDirection d) {
  return d == EvalDirection::Transpose ? HXF_TRANSPOSE : HXF_FORWARD;
}
// a context's staging buffers serve one host-memory call at a time
std::mutex& staging_mutex() {
  static std::mutex mu;
  return mu;
}
}  // namespace

std::vector<int64_t> element_node_indices(const HexMesh& mesh, int64_t e) {
  if (e < 0 || e >= mesh.num_elements())
    throw std::invalid_argument("element_node_indices: element out of range");
  const int p = mesh.p;
  const int64_t ex = e % mesh.dims[0], ey = (e / mesh.dims[0]) % mesh.dims[1];
  const int64_t ez = e / (int64_t(mesh.dims[0]) * mesh.dims[1]);
  const int64_t NX = mesh.nodes_per_axis[0], NY = mesh.nodes_per_axis[1];
  std::vector<int64_t> idx(size_t(mesh.nodes_per_elem()));
  size_t s = 0;
  for (int kz = 0; kz <= p; ++kz)
    for (int ky = 0; ky <= p; ++ky)
      for (int kx = 0; kx <= p; ++kx) idx[s++] = (ex * p + kx) + NX * ((ey * p + ky) + NY * (ez * p + kz));
  return idx;
}

ElemRestriction::ElemRestriction(std::shared_ptr<Device> dev, int p, int m_, int64_t E, int64_t nL,
                                 const int64_t* indices, std::array<int, 3> dims)
    : num_elements(E), elem_size((p + 1) * (p + 1) * (p + 1)), n_L(nL), m(m_), dev_(std::move(dev)) {
  check(hxf_elem_restriction_create(dev_->ctx(), p, m_, E, nL, indices, dims.data(), &r_));
}
ElemRestriction::~ElemRestriction() {
  if (r_) hxf_elem_restriction_destroy(r_);
}
void ElemRestriction::apply_g(std::span<const double> l, std::span<double> e) const {
  std::lock_guard<std::mutex> lock(staging_mutex());
  check(hxf_elem_restriction_apply(r_, 0, l.data(), int64_t(l.size()), e.data(), int64_t(e.size()),
                                   HXF_HOST));
}
void ElemRestriction::apply_g_transpose(std::span<const double> e, std::span<double> l) const {
  std::lock_guard<std::mutex> lock(staging_mutex());
  check(hxf_elem_restriction_apply(r_, 1, e.data(), int64_t(e.size()), l.data(), int64_t(l.size()),
                                   HXF_HOST));
}
std::vector<double> ElemRestriction::multiplicity() const {
  std::vector<double> out(static_cast<size_t>(n_L));
  std::lock_guard<std::mutex> lock(staging_mutex());
  check(hxf_elem_restriction_multiplicity(r_, out.data(), int64_t(out.size()), HXF_HOST));
  return out;
}
void ElemRestriction::gather_scalar(std::span<const double> e, std::span<double> l) const {
  std::lock_guard<std::mutex> lock(staging_mutex());
  check(hxf_elem_restriction_gather_scalar(r_, e.data(), int64_t(e.size()), l.data(),
                                           int64_t(l.size()), HXF_HOST));
}

std::unique_ptr<ElemRestriction> make_restriction(const HexMesh& mesh, int m, int device) {
  if (m < 1) throw std::invalid_argument("make_restriction: m must be >= 1");
  // the structured box: no index table is stored or uploaded (mesh.cpp:80-104)
  return std::make_unique<ElemRestriction>(Device::get(device), mesh.p, m, mesh.num_elements(),
                                           mesh.n_L, nullptr, mesh.dims);
}

void contract_batch(const KernelPlan& plan, std::span<const double> matrix, int n_out, int n_in,
                    int dim, std::array<int, 3> in_shape, int64_t ne, std::span<const double> in,
                    std::span<double> out, bool accumulate) {
  auto dev = Device::get(plan.device);
  uint64_t count = 0;
  {
    std::lock_guard<std::mutex> lock(staging_mutex());
    check(hxf_contract_batch(dev->ctx(), matrix.data(), int64_t(matrix.size()), n_out, n_in, dim,
                             in_shape.data(), ne, in.data(), int64_t(in.size()), out.data(),
                             int64_t(out.size()), accumulate ? 1 : 0, HXF_HOST, &count));
  }
  if (plan.flops) plan.flops->ops.fetch_add(count, std::memory_order_relaxed);
}

void apply_basis_batch(const KernelPlan& plan, const TensorBasis& basis, EvalMode mode,
                       EvalDirection dir, int64_t ne, std::span<const double> in,
                       std::span<double> out) {
  const int64_t nd = basis.num_nodes(), nq = basis.num_qpts();
  const bool grad = mode == EvalMode::Grad, fwd = dir == EvalDirection::Forward;
  const int64_t in_e = fwd ? nd : (grad ? 3 * nq : nq), out_e = fwd ? (grad ? 3 * nq : nq) : nd;
  if (int64_t(in.size()) < ne * in_e || int64_t(out.size()) < ne * out_e)
    throw std::invalid_argument("apply_basis_batch: buffer too small");
  auto dev = Device::get(plan.device);
  {
    std::lock_guard<std::mutex> lock(staging_mutex());
    check(hxf_basis_apply(dev->ctx(), basis.p, basis.q, basis.interp1d.data(), basis.grad1d.data(),
                          mode_of(mode), dir_of(dir), ne, in.data(), out.data(), HXF_HOST));
  }
  if (plan.flops)
    plan.flops->ops.fetch_add(uint64_t(ne) * hxf_flops_estimate(basis.p, basis.q, 1, mode_of(mode)),
                              std::memory_order_relaxed);
}

uint64_t flops_estimate(const KernelPlan& plan, EvalMode mode) {
  return hxf_flops_estimate(plan.p, plan.q, plan.m, mode_of(mode));
}

void apply_tensor_3d(const TensorBasis& basis, EvalMode mode, EvalDirection dir, int m,
                     std::span<const double> u, std::span<double> v, int device) {
  auto dev = Device::get(device);
  std::lock_guard<std::mutex> lock(staging_mutex());
  check(hxf_apply_tensor_3d(dev->ctx(), basis.p, basis.q, basis.interp1d.data(),
                            basis.grad1d.data(), mode_of(mode), dir_of(dir), m, u.data(),
                            int64_t(u.size()), v.data(), int64_t(v.size()), HXF_HOST));
}

}  // namespace hexfem_b200
