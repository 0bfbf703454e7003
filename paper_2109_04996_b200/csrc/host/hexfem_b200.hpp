// Host-side C++ mirror of the reference's (hexfem) BP API, B200-native
// underneath: setup tables are built on the host exactly as the reference
// builds them (so meshes, indices and RHS agree bit for bit), every
// operator-sized computation runs on the GPU through the hxf C-ABI
// (include/hxf.h).  Names follow the reference's public API
// (proj/include/hexfem/*.hpp) so callers switch by namespace.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <span>
#include <atomic>
#include <stdexcept>
#include <string>
#include <vector>

#include "hxf.h"

namespace hexfem_b200 {

// ---- errors: hxf status -> the reference's exception types ----------------
void check(int status);

// ---- quadrature / basis (quadrature.hpp:7-22, tensor_basis.hpp:17-33) ----
enum class QuadratureKind { GaussLegendre, GaussLobattoLegendre };
struct QuadratureRule {
  QuadratureKind kind = QuadratureKind::GaussLegendre;
  int q = 0;
  std::vector<double> points, weights;
};
QuadratureRule make_quadrature(QuadratureKind kind, int q);

struct TensorBasis {
  int p = 0, q = 0;
  std::vector<double> nodes;
  QuadratureRule quad;
  std::vector<double> interp1d, grad1d;  // q x (p+1) row-major
  bool collocated = false;
  int num_nodes() const { return (p + 1) * (p + 1) * (p + 1); }
  int num_qpts() const { return q * q * q; }
};
TensorBasis make_basis(int p, const QuadratureRule& quad);

// ---- mesh (mesh.hpp:9-41) ------------------------------------------------
enum class Deformation { None, Sine };
struct HexMesh {
  std::array<int, 3> dims{};
  int p = 1;
  std::array<int64_t, 3> nodes_per_axis{};
  int64_t n_L = 0;
  std::vector<double> coords;  // 3*n_L component-major (empty: device-built, see mesh_coords)
  std::array<int, 3> global_dims{}, offset{};  // the element box this lattice is part of
  std::vector<int64_t> boundary_nodes;
  Deformation deformation = Deformation::None;
  int64_t num_elements() const { return int64_t(dims[0]) * dims[1] * dims[2]; }
  int nodes_per_elem() const { return (p + 1) * (p + 1) * (p + 1); }
};
HexMesh build_mesh(int nx, int ny, int nz, int p, Deformation deformation = Deformation::None);
// The host coordinates of a mesh whose coordinates were built on the device
// (bp_setup): rebuilt on demand, bit-equal to build_mesh's.
std::vector<double> mesh_coords(const HexMesh& mesh);

// ---- partitioned box (no reference counterpart) -----------
// The global element box is split into a grid of sub-boxes, one per rank,
// rank = cx + gx (cy + gy cz).  Each sub-box keeps its own lexicographic
// node lattice (interface planes duplicated); global_node_ids maps it back to
// the global numbering of build_mesh bit-exactly.
std::array<int, 3> proc_grid(int nranks, std::array<int, 3> global_dims);
struct Subdomain {
  int rank = 0, nranks = 1;
  std::array<int, 3> grid{1, 1, 1}, coord{0, 0, 0}, global_dims{1, 1, 1}, offset{0, 0, 0},
      dims{1, 1, 1};
  std::array<std::array<int, 2>, 3> neighbor{{{-1, -1}, {-1, -1}, {-1, -1}}};
};
Subdomain make_subdomain(std::array<int, 3> global_dims, int nranks, int rank,
                         std::optional<std::array<int, 3>> grid = std::nullopt);
// The sub-box's mesh: coordinates taken from the global lattice (bit-equal),
// boundary_nodes = nodes on the GLOBAL boundary only.
HexMesh build_submesh(const Subdomain& sd, int p, Deformation deformation = Deformation::None);
std::vector<int64_t> global_node_ids(const Subdomain& sd, int p);
// 1 where this sub-box owns the node (not on a low interface plane)
std::vector<uint8_t> owned_nodes(const Subdomain& sd, int p);

// ---- device context -------------------------------------------------------
class Device {
 public:
  explicit Device(int ordinal = 0);
  ~Device();
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;
  hxf_ctx* ctx() const { return ctx_; }
  static std::shared_ptr<Device> get(int ordinal = 0);  // process-wide per ordinal

 private:
  hxf_ctx* ctx_ = nullptr;
};

// Communicator for a partitioned problem (hxf_comm): NCCL with one rank per
// GPU, or an in-process group (one host thread and one context per rank).
class Communicator {
 public:
  static std::string unique_id();  // HXF_COMM_ID_BYTES bytes (rank 0 makes it)
  static std::shared_ptr<Communicator> nccl(int device, int nranks, int rank, const std::string& id);
  static std::vector<std::shared_ptr<Communicator>> group(const std::vector<int>& devices);
  // peer-to-peer mailboxes (hxf_comm_create_p2p), one rank per process:
  // alloc_p2p returns this rank's IPC handle, p2p() opens the gathered handles.
  // (Ranks sharing one process and device would deadlock: a host thread's
  // cudaFree waits for a peer's spinning receive kernel.)
  struct P2pMailbox {
    std::shared_ptr<Device> dev;
    void* base = nullptr;
    std::string handle;  // HXF_COMM_IPC_HANDLE_BYTES
  };
  static P2pMailbox alloc_p2p(int device, int nranks, int64_t cap);
  static std::shared_ptr<Communicator> p2p(const P2pMailbox& mine, int nranks, int rank, int64_t cap,
                                           const std::vector<std::string>& handles);
  ~Communicator();
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  hxf_comm* handle() const { return comm_; }
  int rank() const { return hxf_comm_rank(comm_); }
  int size() const { return hxf_comm_size(comm_); }
  const std::shared_ptr<Device>& device() const { return dev_; }
  double allreduce_sum(double v) const;  // host scalar through the device

 private:
  Communicator() = default;
  std::shared_ptr<Device> dev_;
  std::shared_ptr<hxf_comm_group> group_;
  std::shared_ptr<void> mailbox_;  // p2p: the mailbox this rank owns (freed after the comm)
  hxf_comm* comm_ = nullptr;
};

// Device buffer owned by a Device context.
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(std::shared_ptr<Device> dev, size_t count);
  ~DeviceBuffer();
  DeviceBuffer(DeviceBuffer&& o) noexcept { swap(o); }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    swap(o);
    return *this;
  }
  double* data() const { return ptr_; }
  size_t size() const { return n_; }
  void upload(const double* src, size_t count);
  void download(double* dst, size_t count) const;

 private:
  void swap(DeviceBuffer& o) {
    std::swap(dev_, o.dev_);
    std::swap(ptr_, o.ptr_);
    std::swap(n_, o.n_);
  }
  std::shared_ptr<Device> dev_;
  double* ptr_ = nullptr;
  size_t n_ = 0;
};

// ---- element restriction (restriction.hpp:14-50; mesh.hpp:33-39) ----------
// Node indices of element e, lexicographic x-fastest (mesh.cpp:80-104).
std::vector<int64_t> element_node_indices(const HexMesh& mesh, int64_t e);

// The restriction lives on the device (hxf_restr): for the structured box
// make_restriction builds, G / G^T are computed from the lattice and G^T
// accumulates in the reference's colour-class order (bitwise equal).
class ElemRestriction {
 public:
  ElemRestriction(std::shared_ptr<Device> dev, int p, int m, int64_t num_elements, int64_t n_L,
                  const int64_t* indices, std::array<int, 3> dims);
  ~ElemRestriction();
  ElemRestriction(const ElemRestriction&) = delete;
  ElemRestriction& operator=(const ElemRestriction&) = delete;
  int64_t num_elements = 0;
  int elem_size = 0;
  int64_t n_L = 0;
  int m = 1;
  hxf_restr* handle() const { return r_; }
  void apply_g(std::span<const double> l_vec, std::span<double> e_vec) const;
  void apply_g_transpose(std::span<const double> e_vec, std::span<double> l_vec) const;
  std::vector<double> multiplicity() const;
  void gather_scalar(std::span<const double> e_scalar, std::span<double> l_scalar) const;

 private:
  std::shared_ptr<Device> dev_;
  hxf_restr* r_ = nullptr;
};
std::unique_ptr<ElemRestriction> make_restriction(const HexMesh& mesh, int m, int device = 0);

// ---- contraction kernels / tensor basis (contraction.hpp:13-75,
// tensor_basis.hpp:35-47) on the GPU; bitwise equal to the reference's
// sum-factorized path (KernelPath::Naive is the reference's oracle path).
enum class EvalMode { Interp, Grad };
enum class EvalDirection { Forward, Transpose };
struct FlopCounter {
  std::atomic<uint64_t> ops{0};
  void reset() { ops.store(0); }
  uint64_t count() const { return ops.load(); }
};
struct KernelPlan {
  int p = 1;
  int q = 2;
  int m = 1;
  int block = 8;  // accepted, ignored
  FlopCounter* flops = nullptr;
  int device = 0;
};
void contract_batch(const KernelPlan& plan, std::span<const double> matrix, int n_out, int n_in,
                    int dim, std::array<int, 3> in_shape, int64_t ne, std::span<const double> in,
                    std::span<double> out, bool accumulate = false);
void apply_basis_batch(const KernelPlan& plan, const TensorBasis& basis, EvalMode mode,
                       EvalDirection dir, int64_t ne, std::span<const double> in,
                       std::span<double> out);
uint64_t flops_estimate(const KernelPlan& plan, EvalMode mode);
void apply_tensor_3d(const TensorBasis& basis, EvalMode mode, EvalDirection dir, int m,
                     std::span<const double> u, std::span<double> v, int device = 0);

// ---- BP problems (bench.hpp:16-58) --------------------------------------
enum class BpId { BP1 = 1, BP2, BP3, BP4, BP5, BP6 };
const char* bp_name(BpId bp);
std::optional<BpId> parse_bp(const std::string& name);
int bp_components(BpId bp);
int bp_quadrature_points(BpId bp, int p);
QuadratureKind bp_quadrature_kind(BpId bp);
double bp_alpha(BpId bp);
double bp_beta(BpId bp);
bool bp_has_constraints(BpId bp);
int64_t bp_dof_count(BpId bp, int p, std::array<int, 3> dims);
double manufactured_solution(double x, double y, double z);
double manufactured_rhs(double x, double y, double z);

struct BpConfig {
  BpId bp = BpId::BP1;
  int p = 1;
  std::array<int, 3> dims{1, 1, 1};
  Deformation deformation = Deformation::None;
  int threads = 1;  // accepted for API compatibility; the GPU is the worker
  std::optional<int> fixed_iterations = 20;
  double tol_rel = 1e-8;
  int max_iter = 2000;
  int device = 0;
  // setup fields (coordinates, manufactured f and u, b = B f) on the host (the
  // reference's path; f bit-exact on the sine box too) instead of the device
  bool host_setup = false;
  // partitioned: dims are the GLOBAL element counts, this rank builds its sub-box
  std::shared_ptr<Communicator> comm;
  std::optional<std::array<int, 3>> proc_grid;
};

struct SolveReport {
  int iterations = 0;
  std::vector<double> residual_history;
  bool converged = false;
  double apply_time_seconds = 0.0;  // device time in the operator kernel
  double total_time_seconds = 0.0;  // device time of the whole solve
};

// The operator handle (MatFreeOperator analogue) owns its device data.
class Operator {
 public:
  Operator(std::shared_ptr<Device> dev, const hxf_operator_desc& desc);
  ~Operator();
  Operator(const Operator&) = delete;
  Operator& operator=(const Operator&) = delete;
  hxf_op* handle() const { return op_; }
  int64_t size() const { return size_; }
  void apply_host(const double* x, double* y) const;
  void apply_device(const double* x, double* y, void* stream = nullptr) const;
  void diagonal_device(double* d) const;
  void set_partition(const Communicator& comm, const Subdomain& sd) const;
  SolveReport pcg(const double* b, const double* diag, const hxf_pcg_options& o, double* x,
                  hxf_memspace space) const;
  // pipelined consecutive solves from host vectors (hxf_pcg_host_batch)
  std::vector<SolveReport> pcg_host_batch(const std::vector<const double*>& b, const double* diag,
                                          const hxf_pcg_options& o,
                                          const std::vector<double*>& x) const;

 private:
  std::shared_ptr<Device> dev_;
  hxf_op* op_ = nullptr;
  int64_t size_ = 0;
};

struct BpProblem {
  BpConfig config;
  HexMesh mesh;
  TensorBasis basis;
  int m = 1;
  int64_t n_dofs = 0;
  std::vector<int64_t> constrained;
  std::vector<double> rhs;          // B f, constrained entries zeroed (host copy: host_rhs())
  std::vector<double> exact_nodal;  // nodal interpolant of u* (host copy: host_exact())
  std::shared_ptr<Device> device;
  Subdomain sub;  // whole box unless config.comm is set
  int64_t n_dofs_local = 0;
  std::unique_ptr<Operator> op;
  DeviceBuffer d_rhs, d_diag, d_x, d_b;
  bool diag_ready = false;
  int64_t size() const { return int64_t(m) * mesh.n_L; }
  const double* diagonal_device();  // computed once, cached
  // host copies of the device-built fields, made on first use
  const std::vector<double>& host_rhs();
  const std::vector<double>& host_exact();
  double setup_seconds = 0;  // host wall time of bp_setup
};

std::unique_ptr<BpProblem> bp_setup(const BpConfig& config);

struct BpSolveResult {
  std::vector<double> x;
  SolveReport report;
};
BpSolveResult solve_bp(BpProblem& problem, bool jacobi = true);

// comm: sum the squared error over sub-boxes (partitioned problems)
double l2_error(const HexMesh& mesh, int m, const std::vector<double>& u_h,
                const std::function<double(double, double, double)>& exact,
                std::shared_ptr<Device> dev, const Communicator* comm = nullptr);

struct BenchRecord {
  std::string bp;
  int p = 0, q = 0;
  int64_t E = 0, n = 0;
  int P = 1;
  int iterations = 0;
  double seconds = 0, dofs_rate = 0, n_per_rank = 0;
  double apply_seconds = 0;  // device time in the operator kernel, same rep
};
BenchRecord run_bench(const BpConfig& config);

// Scaling sweeps and record formats (bench.hpp:97-140, bench.cpp:231-381).  P
// is the rank (GPU) count here — the reference's worker-thread count.
struct ScalingRow {
  BenchRecord record;
  double T_1 = 0;  // seconds at P = 1, same problem
  double T_P = 0;
  double eta = 0;  // T_1 / (P T_P)
};
struct ScalingSummary {
  double r_max = 0;                     // max dofs_rate per rank
  std::optional<double> n08_per_rank;   // n/P where eta crosses 0.8 (log-linear)
  double work_constant = 0;             // C of t = C n / (eta P r_max), least squares
};
struct SweepResult {
  std::vector<ScalingRow> rows;  // ascending n/P, then n, then P
  ScalingSummary summary;
};
using TimingModel = std::function<double(int64_t n, int P)>;

// Measured mode runs P = 1 on this process's GPU; P > 1 needs one process per
// GPU (bench.py --gpus P) and is rejected here unless a timing model is given.
SweepResult run_scaling_sweep(BpId bp, int p, const std::vector<std::array<int, 3>>& dims_list,
                              const std::vector<int>& ranks_list, int iterations,
                              Deformation deformation = Deformation::None,
                              const TimingModel& timing_override = {});
// rows -> summary (also usable on records gathered from separate bench runs)
ScalingSummary scaling_summary(std::vector<ScalingRow>& rows);
double time_to_solution(double work_constant, double n, double eta, double P, double r_max);
std::string format_double(double v);  // shortest round-trip form
std::string bench_record_json(const BenchRecord& rec);
std::string sweep_csv_header();
std::string sweep_csv(const SweepResult& result);

// Dense matrix of the operator by applying it to unit vectors on the device
// (the reference's reference_assemble is a dense quadrature loop, oracle only;
// operator.cpp:258-349).  Rejected above 20000 unknowns like the reference.
std::vector<double> assemble_dense(BpProblem& problem);

}  // namespace hexfem_b200
