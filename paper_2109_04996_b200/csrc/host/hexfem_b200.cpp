// Host-side mirror of the reference BP API over the hxf C-ABI.
//
// Setup tables (quadrature, Lagrange basis, mesh lattice, manufactured
// fields) follow the reference formulas and operation order
// (proj/src/quadrature.cpp, tensor_basis.cpp, mesh.cpp, bench.cpp) so the
// node coordinates, restriction numbering and RHS agree with it bit for bit;
// the geometric factors, operator applies, diagonal and PCG run on the GPU.
#include "hexfem_b200.hpp"

#include <chrono>

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <mutex>

namespace hexfem_b200 {

void check(int status) {
  if (status == HXF_OK) return;
  const std::string msg = hxf_last_error();
  if (status == HXF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);  // HXF_ENUMERIC and device failures
}

// ------------------------------------------------------------ quadrature
namespace {
struct Legendre {
  double value, derivative;
};

Legendre legendre_eval(int n, double x) {
  if (n == 0) return {1.0, 0.0};
  double pm1 = 1.0, p = x;
  for (int k = 1; k < n; ++k) {
    const double next = ((2 * k + 1) * x * p - k * pm1) / (k + 1);
    pm1 = p;
    p = next;
  }
  const double denom = x * x - 1.0;
  const double dp = std::abs(denom) > 1e-10
                        ? n * (x * p - pm1) / denom
                        : 0.5 * n * (n + 1) * (x >= 0 ? 1.0 : (n % 2 ? 1.0 : -1.0));
  return {p, dp};
}
}  // namespace

QuadratureRule make_quadrature(QuadratureKind kind, int q) {
  QuadratureRule r;
  r.kind = kind;
  r.q = q;
  r.points.assign(size_t(std::max(q, 0)), 0.0);
  r.weights.assign(size_t(std::max(q, 0)), 0.0);
  if (kind == QuadratureKind::GaussLegendre) {
    if (q < 1)
      throw std::invalid_argument("make_quadrature: Gauss-Legendre needs q >= 1, got " +
                                  std::to_string(q));
    for (int i = 0; i < q / 2; ++i) {
      double x = -std::cos(M_PI * (i + 0.75) / (q + 0.5));
      for (int it = 0; it < 100; ++it) {
        const Legendre L = legendre_eval(q, x);
        const double dx = L.value / L.derivative;
        x -= dx;
        if (std::abs(dx) <= 1e-15) break;
      }
      const double dp = legendre_eval(q, x).derivative;
      const double w = 2.0 / ((1.0 - x * x) * dp * dp);
      r.points[size_t(i)] = x;
      r.weights[size_t(i)] = w;
      r.points[size_t(q - 1 - i)] = -x;
      r.weights[size_t(q - 1 - i)] = w;
    }
    if (q % 2 == 1) {
      const double dp = legendre_eval(q, 0.0).derivative;
      r.points[size_t(q / 2)] = 0.0;
      r.weights[size_t(q / 2)] = 2.0 / (dp * dp);
    }
    return r;
  }
  if (q < 2)
    throw std::invalid_argument("make_quadrature: Gauss-Lobatto-Legendre needs q >= 2, got " +
                                std::to_string(q));
  const int n = q - 1;
  const double end_w = 2.0 / (double(n) * (n + 1));
  r.points[0] = -1.0;
  r.points[size_t(q - 1)] = 1.0;
  r.weights[0] = end_w;
  r.weights[size_t(q - 1)] = end_w;
  for (int i = 1; i < q / 2; ++i) {
    double x = -std::cos(M_PI * i / n);
    for (int it = 0; it < 100; ++it) {
      const Legendre L = legendre_eval(n, x);
      const double d2p = (2.0 * x * L.derivative - double(n) * (n + 1) * L.value) / (1.0 - x * x);
      const double dx = L.derivative / d2p;
      x -= dx;
      if (std::abs(dx) <= 1e-15) break;
    }
    const double pv = legendre_eval(n, x).value;
    const double w = 2.0 / (double(n) * (n + 1) * pv * pv);
    r.points[size_t(i)] = x;
    r.weights[size_t(i)] = w;
    r.points[size_t(q - 1 - i)] = -x;
    r.weights[size_t(q - 1 - i)] = w;
  }
  if (q % 2 == 1) {
    const double pv = legendre_eval(n, 0.0).value;
    r.points[size_t(q / 2)] = 0.0;
    r.weights[size_t(q / 2)] = 2.0 / (double(n) * (n + 1) * pv * pv);
  }
  return r;
}

// ------------------------------------------------------------ basis
namespace {
double lagrange(const std::vector<double>& nd, int j, double x) {
  double r = 1.0;
  for (int m = 0; m < int(nd.size()); ++m)
    if (m != j) r *= (x - nd[size_t(m)]) / (nd[size_t(j)] - nd[size_t(m)]);
  return r;
}
double lagrange_d(const std::vector<double>& nd, int j, double x) {
  double s = 0.0;
  for (int i = 0; i < int(nd.size()); ++i) {
    if (i == j) continue;
    double prod = 1.0;
    for (int m = 0; m < int(nd.size()); ++m)
      if (m != i && m != j) prod *= (x - nd[size_t(m)]) / (nd[size_t(j)] - nd[size_t(m)]);
    s += prod / (nd[size_t(j)] - nd[size_t(i)]);
  }
  return s;
}
}  // namespace

TensorBasis make_basis(int p, const QuadratureRule& quad) {
  if (p < 1) throw std::invalid_argument("make_basis: p must be >= 1, got " + std::to_string(p));
  if (quad.q < 1 || int(quad.points.size()) != quad.q)
    throw std::invalid_argument("make_basis: invalid quadrature rule");
  TensorBasis b;
  b.p = p;
  b.q = quad.q;
  b.quad = quad;
  b.nodes = make_quadrature(QuadratureKind::GaussLobattoLegendre, p + 1).points;
  b.collocated = quad.kind == QuadratureKind::GaussLobattoLegendre && quad.q == p + 1;
  const int n1 = p + 1;
  b.interp1d.assign(size_t(quad.q) * n1, 0.0);
  b.grad1d.assign(size_t(quad.q) * n1, 0.0);
  for (int iq = 0; iq < quad.q; ++iq)
    for (int j = 0; j < n1; ++j) {
      b.interp1d[size_t(iq) * n1 + j] = lagrange(b.nodes, j, quad.points[size_t(iq)]);
      b.grad1d[size_t(iq) * n1 + j] = lagrange_d(b.nodes, j, quad.points[size_t(iq)]);
    }
  return b;
}

// ------------------------------------------------------------ mesh
namespace {
// The lattice of the element sub-box [off, off + loc) of a global box of
// `glob` elements, coordinates evaluated on the global 1-D axes (mesh.cpp:
// 42-78) so a sub-box mesh is bit-equal to the matching part of the global.
HexMesh build_box_mesh(std::array<int, 3> glob, std::array<int, 3> off, std::array<int, 3> loc,
                       int p, Deformation deformation, bool with_coords = true) {
  HexMesh mesh;
  mesh.dims = loc;
  mesh.global_dims = glob;
  mesh.offset = off;
  mesh.p = p;
  mesh.deformation = deformation;
  mesh.nodes_per_axis = {int64_t(loc[0]) * p + 1, int64_t(loc[1]) * p + 1, int64_t(loc[2]) * p + 1};
  mesh.n_L = mesh.nodes_per_axis[0] * mesh.nodes_per_axis[1] * mesh.nodes_per_axis[2];
  const std::vector<double> gll = make_quadrature(QuadratureKind::GaussLobattoLegendre, p + 1).points;
  auto axis = [&](int ne) {
    std::vector<double> c(size_t(ne) * p + 1);
    const double h = 1.0 / ne;
    for (int k = 0; k < ne; ++k)
      for (int j = 0; j <= p; ++j) c[size_t(k) * p + size_t(j)] = (k + 0.5 * (gll[size_t(j)] + 1.0)) * h;
    c.back() = 1.0;
    c.front() = 0.0;
    return c;
  };
  const auto cx = axis(glob[0]), cy = axis(glob[1]), cz = axis(glob[2]);
  const int64_t NX = mesh.nodes_per_axis[0], NY = mesh.nodes_per_axis[1],
                NZ = mesh.nodes_per_axis[2];
  const int64_t GX = int64_t(glob[0]) * p + 1, GY = int64_t(glob[1]) * p + 1,
                GZ = int64_t(glob[2]) * p + 1;
  const int64_t ox = int64_t(off[0]) * p, oy = int64_t(off[1]) * p, oz = int64_t(off[2]) * p;
  if (!with_coords) {  // topology only: the global-boundary nodes (mesh.cpp:67-71)
    for (int64_t iz = 0; iz < NZ; ++iz)
      for (int64_t iy = 0; iy < NY; ++iy)
        for (int64_t ix = 0; ix < NX; ++ix) {
          const int64_t gx = ox + ix, gy = oy + iy, gz = oz + iz;
          if (gx == 0 || gx == GX - 1 || gy == 0 || gy == GY - 1 || gz == 0 || gz == GZ - 1)
            mesh.boundary_nodes.push_back(ix + NX * (iy + NY * iz));
        }
    return mesh;
  }
  mesh.coords.assign(size_t(3 * mesh.n_L), 0.0);
  // the sine bump factorises: s(x,y,z) = sin(pi x) sin(pi y) sin(pi z), with
  // the reference's evaluation order ((eps*sx)*sy)*sz kept per node
  std::vector<double> sx(cx.size()), sy(cy.size()), sz(cz.size());
  for (size_t i = 0; i < cx.size(); ++i) sx[i] = std::sin(M_PI * cx[i]);
  for (size_t i = 0; i < cy.size(); ++i) sy[i] = std::sin(M_PI * cy[i]);
  for (size_t i = 0; i < cz.size(); ++i) sz[i] = std::sin(M_PI * cz[i]);
  int64_t node = 0;
  for (int64_t iz = 0; iz < NZ; ++iz)
    for (int64_t iy = 0; iy < NY; ++iy)
      for (int64_t ix = 0; ix < NX; ++ix, ++node) {
        const size_t gx = size_t(ox + ix), gy = size_t(oy + iy), gz = size_t(oz + iz);
        double x = cx[gx], y = cy[gy], z = cz[gz];
        if (deformation == Deformation::Sine) {
          const double bump = 0.05 * sx[gx] * sy[gy] * sz[gz];
          x += bump;
          y += bump;
          z += bump;
        }
        mesh.coords[size_t(node)] = x;
        mesh.coords[size_t(mesh.n_L + node)] = y;
        mesh.coords[size_t(2 * mesh.n_L + node)] = z;
        if (gx == 0 || int64_t(gx) == GX - 1 || gy == 0 || int64_t(gy) == GY - 1 || gz == 0 ||
            int64_t(gz) == GZ - 1)
          mesh.boundary_nodes.push_back(node);
      }
  return mesh;
}
}  // namespace

HexMesh build_mesh(int nx, int ny, int nz, int p, Deformation deformation) {
  if (nx < 1 || ny < 1 || nz < 1)
    throw std::invalid_argument("build_mesh: element counts must be >= 1");
  if (p < 1) throw std::invalid_argument("build_mesh: p must be >= 1");
  return build_box_mesh({nx, ny, nz}, {0, 0, 0}, {nx, ny, nz}, p, deformation);
}

std::vector<double> mesh_coords(const HexMesh& mesh) {
  if (!mesh.coords.empty()) return mesh.coords;
  return build_box_mesh(mesh.global_dims, mesh.offset, mesh.dims, mesh.p, mesh.deformation).coords;
}

// ------------------------------------------------------------ partition
std::array<int, 3> proc_grid(int nranks, std::array<int, 3> global_dims) {
  if (nranks < 1) throw std::invalid_argument("proc_grid: nranks must be >= 1");
  // prime factors, largest first, each onto the axis with the most elements
  // per rank (ties: x, then y, then z): 2 -> 2x1x1, 4 -> 2x2x1, 8 -> 2x2x2
  std::vector<int> f;
  for (int n = nranks, d = 2; n > 1;) {
    if (n % d == 0) {
      f.push_back(d);
      n /= d;
    } else {
      ++d;
    }
  }
  std::sort(f.rbegin(), f.rend());
  std::array<int, 3> g{1, 1, 1};
  for (int k : f) {
    int best = 0;
    for (int a = 1; a < 3; ++a)
      if (double(global_dims[size_t(a)]) / g[size_t(a)] >
          double(global_dims[size_t(best)]) / g[size_t(best)])
        best = a;
    g[size_t(best)] *= k;
  }
  return g;
}

Subdomain make_subdomain(std::array<int, 3> global_dims, int nranks, int rank,
                         std::optional<std::array<int, 3>> grid) {
  if (rank < 0 || rank >= nranks) throw std::invalid_argument("make_subdomain: bad rank");
  Subdomain sd;
  sd.rank = rank;
  sd.nranks = nranks;
  sd.global_dims = global_dims;
  sd.grid = grid ? *grid : proc_grid(nranks, global_dims);
  if (sd.grid[0] * sd.grid[1] * sd.grid[2] != nranks)
    throw std::invalid_argument("make_subdomain: process grid does not match the rank count");
  sd.coord = {rank % sd.grid[0], (rank / sd.grid[0]) % sd.grid[1], rank / (sd.grid[0] * sd.grid[1])};
  for (size_t a = 0; a < 3; ++a) {
    const int G = global_dims[a], g = sd.grid[a], c = sd.coord[a];
    if (G < g) throw std::invalid_argument("make_subdomain: fewer elements than ranks along an axis");
    const int base = G / g, extra = G % g;
    sd.dims[a] = base + (c < extra ? 1 : 0);
    sd.offset[a] = c * base + std::min(c, extra);
    std::array<int, 3> lo = sd.coord, hi = sd.coord;
    lo[a] -= 1;
    hi[a] += 1;
    auto rank_of = [&](const std::array<int, 3>& k) {
      return k[0] + sd.grid[0] * (k[1] + sd.grid[1] * k[2]);
    };
    sd.neighbor[a][0] = c > 0 ? rank_of(lo) : -1;
    sd.neighbor[a][1] = c + 1 < g ? rank_of(hi) : -1;
  }
  return sd;
}

HexMesh build_submesh(const Subdomain& sd, int p, Deformation deformation) {
  if (p < 1) throw std::invalid_argument("build_mesh: p must be >= 1");
  return build_box_mesh(sd.global_dims, sd.offset, sd.dims, p, deformation);
}

std::vector<int64_t> global_node_ids(const Subdomain& sd, int p) {
  const int64_t NX = int64_t(sd.dims[0]) * p + 1, NY = int64_t(sd.dims[1]) * p + 1,
                NZ = int64_t(sd.dims[2]) * p + 1;
  const int64_t GX = int64_t(sd.global_dims[0]) * p + 1, GY = int64_t(sd.global_dims[1]) * p + 1;
  std::vector<int64_t> ids(size_t(NX * NY * NZ));
  size_t i = 0;
  for (int64_t iz = 0; iz < NZ; ++iz)
    for (int64_t iy = 0; iy < NY; ++iy)
      for (int64_t ix = 0; ix < NX; ++ix)
        ids[i++] = (int64_t(sd.offset[0]) * p + ix) +
                   GX * ((int64_t(sd.offset[1]) * p + iy) + GY * (int64_t(sd.offset[2]) * p + iz));
  return ids;
}

std::vector<uint8_t> owned_nodes(const Subdomain& sd, int p) {
  const int64_t NX = int64_t(sd.dims[0]) * p + 1, NY = int64_t(sd.dims[1]) * p + 1,
                NZ = int64_t(sd.dims[2]) * p + 1;
  const bool lx = sd.neighbor[0][0] >= 0, ly = sd.neighbor[1][0] >= 0, lz = sd.neighbor[2][0] >= 0;
  std::vector<uint8_t> own(size_t(NX * NY * NZ));
  size_t i = 0;
  for (int64_t iz = 0; iz < NZ; ++iz)
    for (int64_t iy = 0; iy < NY; ++iy)
      for (int64_t ix = 0; ix < NX; ++ix)
        own[i++] = !((lx && ix == 0) || (ly && iy == 0) || (lz && iz == 0));
  return own;
}

// ------------------------------------------------------------ device
Device::Device(int ordinal) { check(hxf_context_create(ordinal, nullptr, &ctx_)); }
Device::~Device() {
  if (ctx_) hxf_context_destroy(ctx_);
}
std::shared_ptr<Device> Device::get(int ordinal) {
  static std::mutex mu;
  static std::map<int, std::weak_ptr<Device>> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto sp = cache[ordinal].lock();
  if (!sp) {
    sp = std::make_shared<Device>(ordinal);
    cache[ordinal] = sp;
  }
  return sp;
}

DeviceBuffer::DeviceBuffer(std::shared_ptr<Device> dev, size_t count) : dev_(std::move(dev)), n_(count) {
  void* p = nullptr;
  check(hxf_malloc(dev_->ctx(), uint64_t(count) * 8, &p));
  ptr_ = static_cast<double*>(p);
}
DeviceBuffer::~DeviceBuffer() {
  if (ptr_ && dev_) hxf_free(dev_->ctx(), ptr_);
}
void DeviceBuffer::upload(const double* src, size_t count) {
  check(hxf_memcpy(dev_->ctx(), ptr_, src, uint64_t(count) * 8, 0));
}
void DeviceBuffer::download(double* dst, size_t count) const {
  check(hxf_memcpy(dev_->ctx(), dst, ptr_, uint64_t(count) * 8, 1));
}

std::string Communicator::unique_id() {
  std::string id(HXF_COMM_ID_BYTES, '\0');
  check(hxf_comm_unique_id(reinterpret_cast<unsigned char*>(id.data())));
  return id;
}
std::shared_ptr<Communicator> Communicator::nccl(int device, int nranks, int rank,
                                                 const std::string& id) {
  if (id.size() != HXF_COMM_ID_BYTES) throw std::invalid_argument("nccl: bad unique id length");
  std::shared_ptr<Communicator> c(new Communicator());
  c->dev_ = Device::get(device);
  check(hxf_comm_create_nccl(c->dev_->ctx(), nranks, rank,
                             reinterpret_cast<const unsigned char*>(id.data()), &c->comm_));
  return c;
}
std::vector<std::shared_ptr<Communicator>> Communicator::group(const std::vector<int>& devices) {
  hxf_comm_group* g = nullptr;
  check(hxf_comm_group_create(int(devices.size()), &g));
  std::shared_ptr<hxf_comm_group> shared(g, [](hxf_comm_group* p) { hxf_comm_group_destroy(p); });
  std::vector<std::shared_ptr<Communicator>> out;
  for (size_t r = 0; r < devices.size(); ++r) {
    std::shared_ptr<Communicator> c(new Communicator());
    c->dev_ = std::make_shared<Device>(devices[r]);  // own context + stream per sub-domain
    c->group_ = shared;
    check(hxf_comm_create_group(c->dev_->ctx(), g, int(r), &c->comm_));
    out.push_back(c);
  }
  return out;
}
Communicator::P2pMailbox Communicator::alloc_p2p(int device, int nranks, int64_t cap) {
  P2pMailbox m;
  m.dev = Device::get(device);
  m.handle.assign(HXF_COMM_IPC_HANDLE_BYTES, '\0');
  check(hxf_comm_p2p_alloc(m.dev->ctx(), nranks, cap, &m.base,
                           reinterpret_cast<unsigned char*>(m.handle.data())));
  return m;
}

std::shared_ptr<Communicator> Communicator::p2p(const P2pMailbox& mine, int nranks, int rank,
                                                int64_t cap, const std::vector<std::string>& handles) {
  if (int(handles.size()) != nranks) throw std::invalid_argument("p2p: one handle per rank");
  std::string all;
  for (const auto& hd : handles) {
    if (hd.size() != HXF_COMM_IPC_HANDLE_BYTES) throw std::invalid_argument("p2p: bad handle");
    all += hd;
  }
  std::vector<void*> bases(size_t(nranks), nullptr);
  bases[size_t(rank)] = mine.base;
  std::shared_ptr<Communicator> c(new Communicator());
  c->dev_ = mine.dev;
  auto dev = mine.dev;
  c->mailbox_ = std::shared_ptr<void>(mine.base, [dev](void* p) { hxf_comm_p2p_free(dev->ctx(), p); });
  check(hxf_comm_create_p2p(c->dev_->ctx(), nranks, rank, cap, bases.data(),
                            reinterpret_cast<const unsigned char*>(all.data()), &c->comm_));
  return c;
}

Communicator::~Communicator() {
  if (comm_) hxf_comm_destroy(comm_);
  comm_ = nullptr;
  mailbox_.reset();  // after the communicator that used it
}
double Communicator::allreduce_sum(double v) const {
  DeviceBuffer b(dev_, 1);
  b.upload(&v, 1);
  check(hxf_comm_allreduce_sum(comm_, b.data(), 1, nullptr));
  b.download(&v, 1);
  return v;
}

Operator::Operator(std::shared_ptr<Device> dev, const hxf_operator_desc& desc) : dev_(std::move(dev)) {
  check(hxf_operator_create(dev_->ctx(), &desc, &op_));
  size_ = hxf_operator_size(op_);
}
Operator::~Operator() {
  if (op_) hxf_operator_destroy(op_);
}
void Operator::apply_host(const double* x, double* y) const {
  check(hxf_operator_apply(op_, x, y, HXF_HOST, nullptr));
}
void Operator::apply_device(const double* x, double* y, void* stream) const {
  check(hxf_operator_apply(op_, x, y, HXF_DEVICE, stream));
}
void Operator::diagonal_device(double* d) const { check(hxf_operator_diagonal(op_, d, HXF_DEVICE)); }
void Operator::set_partition(const Communicator& comm, const Subdomain& sd) const {
  hxf_partition_desc d{};
  for (int a = 0; a < 3; ++a)
    for (int s = 0; s < 2; ++s) d.neighbor[a][s] = sd.neighbor[size_t(a)][size_t(s)];
  check(hxf_operator_set_partition(op_, comm.handle(), &d));
}

SolveReport Operator::pcg(const double* b, const double* diag, const hxf_pcg_options& o, double* x,
                          hxf_memspace space) const {
  const int cap = (o.fixed_iterations >= 0 ? o.fixed_iterations : o.max_iter) + 2;
  std::vector<double> hist(size_t(std::max(cap, 1)));
  hxf_solve_report rep{};
  rep.residual_history = hist.data();
  rep.history_capacity = cap;
  check(hxf_pcg(op_, b, diag, &o, x, space, &rep));
  SolveReport out;
  out.iterations = rep.iterations;
  out.converged = rep.converged != 0;
  out.residual_history.assign(hist.begin(), hist.begin() + std::min(cap, rep.iterations + 1));
  out.apply_time_seconds = rep.apply_time_seconds;
  out.total_time_seconds = rep.total_time_seconds;
  return out;
}

std::vector<SolveReport> Operator::pcg_host_batch(const std::vector<const double*>& b,
                                                  const double* diag, const hxf_pcg_options& o,
                                                  const std::vector<double*>& x) const {
  if (b.size() != x.size()) throw std::invalid_argument("pcg_host_batch: b / x count mismatch");
  const int cap = (o.fixed_iterations >= 0 ? o.fixed_iterations : o.max_iter) + 2;
  std::vector<std::vector<double>> hist(b.size(), std::vector<double>(size_t(std::max(cap, 1))));
  std::vector<hxf_solve_report> rep(b.size());
  for (size_t k = 0; k < b.size(); ++k) {
    rep[k].residual_history = hist[k].data();
    rep[k].history_capacity = cap;
  }
  check(hxf_pcg_host_batch(op_, int(b.size()), b.data(), diag, &o, x.data(), rep.data()));
  std::vector<SolveReport> out(b.size());
  for (size_t k = 0; k < b.size(); ++k) {
    out[k].iterations = rep[k].iterations;
    out[k].converged = rep[k].converged != 0;
    out[k].residual_history.assign(hist[k].begin(),
                                   hist[k].begin() + std::min(cap, rep[k].iterations + 1));
    out[k].total_time_seconds = rep[k].total_time_seconds;
  }
  return out;
}

// ------------------------------------------------------------ BP tables
const char* bp_name(BpId bp) {
  static const char* names[] = {"?", "bp1", "bp2", "bp3", "bp4", "bp5", "bp6"};
  const int i = int(bp);
  return (i >= 1 && i <= 6) ? names[i] : "?";
}
std::optional<BpId> parse_bp(const std::string& name) {
  for (int i = 1; i <= 6; ++i)
    if (name == bp_name(BpId(i))) return BpId(i);
  return std::nullopt;
}
int bp_components(BpId bp) { return int(bp) % 2 == 1 ? 1 : 3; }
int bp_quadrature_points(BpId bp, int p) { return int(bp) <= 4 ? p + 2 : p + 1; }
QuadratureKind bp_quadrature_kind(BpId bp) {
  return int(bp) <= 4 ? QuadratureKind::GaussLegendre : QuadratureKind::GaussLobattoLegendre;
}
double bp_alpha(BpId bp) { return int(bp) <= 2 ? 0.0 : 1.0; }
double bp_beta(BpId bp) { return int(bp) <= 2 ? 1.0 : 0.0; }
bool bp_has_constraints(BpId bp) { return int(bp) >= 3; }
int64_t bp_dof_count(BpId bp, int p, std::array<int, 3> dims) {
  int64_t count = 1;
  for (int d = 0; d < 3; ++d) {
    const int64_t axis = int64_t(dims[size_t(d)]) * p + 1;
    count *= bp_has_constraints(bp) ? axis - 2 : axis;
  }
  return count * bp_components(bp);
}
double manufactured_solution(double x, double y, double z) {
  return std::sin(M_PI * x) * std::sin(M_PI * y) * std::sin(M_PI * z);
}
double manufactured_rhs(double x, double y, double z) {
  return 3.0 * M_PI * M_PI * manufactured_solution(x, y, z);
}

namespace {
hxf_operator_desc base_desc(const HexMesh& mesh, const TensorBasis& basis, int m) {
  hxf_operator_desc d{};
  d.p = basis.p;
  d.q = basis.q;
  d.m = m;
  d.num_elements = mesh.num_elements();
  d.n_L = mesh.n_L;
  d.interp1d = basis.interp1d.data();
  d.grad1d = basis.grad1d.data();
  d.qpoints = basis.quad.points.data();
  d.indices = nullptr;  // structured box: G from the lattice (mesh.cpp:80-104)
  d.dims[0] = mesh.dims[0];
  d.dims[1] = mesh.dims[1];
  d.dims[2] = mesh.dims[2];
  d.qdata_space = HXF_DEVICE;
  d.block = 8;
  return d;
}

DeviceBuffer device_qdata(const std::shared_ptr<Device>& dev, const HexMesh& mesh,
                          const TensorBasis& basis, const DeviceBuffer& d_coords,
                          hxf_qdata_kind kind) {
  const size_t n = size_t(mesh.num_elements()) * (kind == HXF_QDATA_MASS ? 1 : 6) * basis.num_qpts();
  DeviceBuffer out(dev, n);
  check(hxf_qdata_compute(dev->ctx(), basis.p, basis.q, basis.interp1d.data(), basis.grad1d.data(),
                          basis.quad.weights.data(), mesh.num_elements(), mesh.n_L,
                          d_coords.data(), nullptr, mesh.dims.data(), kind, out.data(),
                          HXF_DEVICE));
  return out;
}
}  // namespace

const double* BpProblem::diagonal_device() {
  if (!diag_ready) {
    op->diagonal_device(d_diag.data());
    diag_ready = true;
  }
  return d_diag.data();
}

// bp_setup (bench.cpp:64-119): mesh + basis on the host, geometric factors,
// RHS mass apply and everything after on the GPU.
const std::vector<double>& BpProblem::host_rhs() {
  if (rhs.size() != size_t(size())) {
    rhs.assign(size_t(size()), 0.0);
    d_rhs.download(rhs.data(), rhs.size());
  }
  return rhs;
}

const std::vector<double>& BpProblem::host_exact() {
  if (exact_nodal.size() != size_t(size())) {
    exact_nodal.assign(size_t(size()), 0.0);
    const auto gll = make_quadrature(QuadratureKind::GaussLobattoLegendre, config.p + 1).points;
    check(hxf_box_fields(device->ctx(), sub.global_dims.data(), sub.offset.data(), sub.dims.data(),
                         config.p, gll.data(), config.deformation == Deformation::Sine ? 1 : 0, m,
                         0, nullptr, nullptr, exact_nodal.data(), HXF_HOST));
  }
  return exact_nodal;
}

std::unique_ptr<BpProblem> bp_setup(const BpConfig& config) {
  const auto t_start = std::chrono::steady_clock::now();
  if (config.p < 1) throw std::invalid_argument("bp_setup: p must be >= 1");
  for (int d : config.dims)
    if (d < 1) throw std::invalid_argument("bp_setup: element counts must be >= 1");
  auto prob = std::make_unique<BpProblem>();
  prob->config = config;
  prob->m = bp_components(config.bp);
  const Communicator* comm = config.comm.get();
  prob->device = comm ? comm->device() : Device::get(config.device);
  auto& dev = prob->device;
  const int q = bp_quadrature_points(config.bp, config.p);
  if (comm) {
    prob->sub = make_subdomain(config.dims, comm->size(), comm->rank(), config.proc_grid);
  } else {
    prob->sub = make_subdomain(config.dims, 1, 0);
  }
  // device setup: the host keeps only the lattice topology (boundary nodes)
  prob->mesh = build_box_mesh(prob->sub.global_dims, prob->sub.offset, prob->sub.dims, config.p,
                              config.deformation, config.host_setup);
  prob->basis = make_basis(config.p, make_quadrature(bp_quadrature_kind(config.bp), q));
  const HexMesh& mesh = prob->mesh;
  const int64_t n_L = mesh.n_L;
  const int m = prob->m;
  const double alpha = bp_alpha(config.bp), beta = bp_beta(config.bp);

  const bool poisson = alpha > 0;
  DeviceBuffer d_coords(dev, size_t(3 * n_L));
  DeviceBuffer d_f(dev, size_t(m) * n_L);
  if (config.host_setup) {
    // the reference's order on the host (mesh.cpp:42-78, bench.cpp:89-105)
    d_coords.upload(mesh.coords.data(), size_t(3 * n_L));
    std::vector<double> f(size_t(m) * n_L);
    prob->exact_nodal.assign(size_t(m) * n_L, 0.0);
    for (int64_t i = 0; i < n_L; ++i) {
      const double x = mesh.coords[size_t(i)], y = mesh.coords[size_t(n_L + i)],
                   z = mesh.coords[size_t(2 * n_L + i)];
      const double u = manufactured_solution(x, y, z);
      const double fv = poisson ? manufactured_rhs(x, y, z) : u;
      for (int c = 0; c < m; ++c) {
        f[size_t(c * n_L + i)] = fv;
        prob->exact_nodal[size_t(c * n_L + i)] = u;
      }
    }
    d_f.upload(f.data(), f.size());
  } else {
    // device: only the 1-D axes cross the bus (hxf_box_fields)
    const auto gll = make_quadrature(QuadratureKind::GaussLobattoLegendre, config.p + 1).points;
    check(hxf_box_fields(dev->ctx(), prob->sub.global_dims.data(), prob->sub.offset.data(),
                         prob->sub.dims.data(), config.p, gll.data(),
                         config.deformation == Deformation::Sine ? 1 : 0, m, poisson ? 1 : 0,
                         d_coords.data(), d_f.data(), nullptr, HXF_DEVICE));
  }
  DeviceBuffer mass_qd = device_qdata(dev, mesh, prob->basis, d_coords, HXF_QDATA_MASS);
  DeviceBuffer diff_qd;
  if (alpha > 0) diff_qd = device_qdata(dev, mesh, prob->basis, d_coords, HXF_QDATA_DIFFUSION);
  d_coords = DeviceBuffer();

  if (bp_has_constraints(config.bp)) prob->constrained = mesh.boundary_nodes;

  // b = B f with the unconstrained mass operator (assembled across interfaces),
  // constrained entries then zeroed (bench.cpp:106-111), all on the device
  prob->d_rhs = DeviceBuffer(dev, size_t(m) * n_L);
  {
    hxf_operator_desc d = base_desc(mesh, prob->basis, m);
    d.mass_qdata = mass_qd.data();
    d.beta = 1.0;
    Operator mass_op(dev, d);
    if (comm) mass_op.set_partition(*comm, prob->sub);
    mass_op.apply_device(d_f.data(), prob->d_rhs.data());
  }
  d_f = DeviceBuffer();

  hxf_operator_desc d = base_desc(mesh, prob->basis, m);
  d.alpha = alpha;
  d.beta = beta;
  d.mass_qdata = beta > 0 ? mass_qd.data() : nullptr;
  d.diff_qdata = alpha > 0 ? diff_qd.data() : nullptr;
  d.constrained = prob->constrained.data();
  d.n_constrained = int64_t(prob->constrained.size());
  prob->op = std::make_unique<Operator>(dev, d);
  if (comm) prob->op->set_partition(*comm, prob->sub);
  prob->n_dofs_local = int64_t(m) * (n_L - int64_t(prob->constrained.size()));
  prob->n_dofs = bp_dof_count(config.bp, config.p, config.dims);  // global
  if (!prob->constrained.empty())
    check(hxf_operator_set_constrained(prob->op->handle(), prob->d_rhs.data(), 0.0, HXF_DEVICE));
  prob->d_diag = DeviceBuffer(dev, size_t(m) * n_L);
  prob->d_x = DeviceBuffer(dev, size_t(m) * n_L);
  prob->setup_seconds =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  return prob;
}

// solve_bp (bench.cpp:121-137), device resident.
BpSolveResult solve_bp(BpProblem& problem, bool jacobi) {
  hxf_pcg_options o{};
  o.tol_rel = problem.config.tol_rel;
  o.max_iter = problem.config.max_iter;
  o.fixed_iterations = problem.config.fixed_iterations ? *problem.config.fixed_iterations : -1;
  o.time_apply = 1;  // SolveReport::apply_time_seconds, as the reference reports it
  const double* diag = jacobi ? problem.diagonal_device() : nullptr;
  BpSolveResult res;
  res.report = problem.op->pcg(problem.d_rhs.data(), diag, o, problem.d_x.data(), HXF_DEVICE);
  res.x.resize(size_t(problem.size()));
  problem.d_x.download(res.x.data(), res.x.size());
  return res;
}

// l2_error (bench.cpp:139-189): Gauss q=p+2 rule, element-wise interpolation.
double l2_error(const HexMesh& mesh, int m, const std::vector<double>& u_h,
                const std::function<double(double, double, double)>& exact,
                std::shared_ptr<Device> dev, const Communicator* comm) {
  const int p = mesh.p, n1 = p + 1, q = p + 2;
  const TensorBasis eb = make_basis(p, make_quadrature(QuadratureKind::GaussLegendre, q));
  const int64_t E = mesh.num_elements(), n_L = mesh.n_L;
  const int S = n1 * n1 * n1, nq = q * q * q;
  if (int64_t(u_h.size()) != int64_t(m) * n_L)
    throw std::invalid_argument("l2_error: solution length mismatch");
  const std::vector<double> coords = mesh_coords(mesh);
  // w det J at the Gauss points on the device
  std::vector<double> wdet(size_t(E) * nq);
  check(hxf_qdata_compute(dev->ctx(), p, q, eb.interp1d.data(), eb.grad1d.data(),
                          eb.quad.weights.data(), E, n_L, coords.data(), nullptr,
                          mesh.dims.data(), HXF_QDATA_MASS, wdet.data(), HXF_HOST));
  // element values of coords (3) and solution (m) -> quadrature points
  const int nfield = 3 + m;
  std::vector<double> ev(size_t(nfield) * E * S);
  const int64_t NX = mesh.nodes_per_axis[0], NY = mesh.nodes_per_axis[1];
  for (int64_t e = 0; e < E; ++e) {
    const int64_t ex = e % mesh.dims[0], ey = (e / mesh.dims[0]) % mesh.dims[1],
                  ez = e / (int64_t(mesh.dims[0]) * mesh.dims[1]);
    int s = 0;
    for (int kz = 0; kz <= p; ++kz)
      for (int ky = 0; ky <= p; ++ky)
        for (int kx = 0; kx <= p; ++kx, ++s) {
          const int64_t node = (ex * p + kx) + NX * ((ey * p + ky) + NY * (ez * p + kz));
          for (int a = 0; a < 3; ++a)
            ev[size_t((a * E + e) * S + s)] = coords[size_t(a * n_L + node)];
          for (int c = 0; c < m; ++c)
            ev[size_t(((3 + c) * E + e) * S + s)] = u_h[size_t(c * n_L + node)];
        }
  }
  std::vector<double> qv(size_t(nfield) * E * nq);
  check(hxf_basis_apply(dev->ctx(), p, q, eb.interp1d.data(), eb.grad1d.data(), HXF_INTERP,
                        HXF_FORWARD, nfield * E, ev.data(), qv.data(), HXF_HOST));
  double err2 = 0.0;
  std::vector<double> diff2(static_cast<size_t>(nq));
  for (int64_t e = 0; e < E; ++e) {
    std::fill(diff2.begin(), diff2.end(), 0.0);
    const double* xq = qv.data() + size_t(e) * nq;
    const double* yq = qv.data() + size_t(E + e) * nq;
    const double* zq = qv.data() + size_t(2 * E + e) * nq;
    for (int c = 0; c < m; ++c) {
      const double* uq = qv.data() + size_t((3 + c) * E + e) * nq;
      for (int i = 0; i < nq; ++i) {
        const double dlt = uq[i] - exact(xq[i], yq[i], zq[i]);
        diff2[size_t(i)] += dlt * dlt;
      }
    }
    for (int i = 0; i < nq; ++i) err2 += wdet[size_t(e * nq + i)] * diff2[size_t(i)];
  }
  if (comm) err2 = comm->allreduce_sum(err2);
  return std::sqrt(err2);
}

// run_bench (bench.cpp:191-229): setup and diagonal untimed; the CG loop is
// repeated 3 times in bench mode and the minimum (device) time recorded.
BenchRecord run_bench(const BpConfig& config) {
  if (config.threads < 1) throw std::invalid_argument("run_bench: threads must be >= 1");
  auto prob = bp_setup(config);
  const double* diag = prob->diagonal_device();
  hxf_pcg_options o{};
  o.tol_rel = config.tol_rel;
  o.max_iter = config.max_iter;
  o.fixed_iterations = config.fixed_iterations ? *config.fixed_iterations : -1;
  // the CG loop timed un-instrumented (min of 3, bench.cpp:206-215), then one
  // solve with per-apply CUDA events for apply_seconds
  const int reps = config.fixed_iterations ? 3 : 1;
  double seconds = std::numeric_limits<double>::infinity(), apply_s = 0;
  int iterations = 0;
  for (int rep = 0; rep < reps; ++rep) {
    const SolveReport r = prob->op->pcg(prob->d_rhs.data(), diag, o, prob->d_x.data(), HXF_DEVICE);
    seconds = std::min(seconds, r.total_time_seconds);
    iterations = r.iterations;
  }
  o.time_apply = 1;
  apply_s = prob->op->pcg(prob->d_rhs.data(), diag, o, prob->d_x.data(), HXF_DEVICE).apply_time_seconds;
  BenchRecord rec;
  rec.bp = bp_name(config.bp);
  rec.p = config.p;
  rec.q = prob->basis.q;
  rec.E = prob->mesh.num_elements();
  rec.n = prob->n_dofs;
  rec.P = config.comm ? config.comm->size() : config.threads;
  rec.iterations = iterations;
  rec.seconds = seconds;
  rec.dofs_rate = double(rec.n) * rec.iterations / rec.seconds;
  rec.n_per_rank = double(rec.n) / rec.P;
  rec.apply_seconds = apply_s;
  return rec;
}

// ---------------------------------------------------------------- sweeps
// (bench.cpp:231-330: the same grouping, ordering and efficiency algebra)
SweepResult run_scaling_sweep(BpId bp, int p, const std::vector<std::array<int, 3>>& dims_list,
                              const std::vector<int>& ranks_list, int iterations,
                              Deformation deformation, const TimingModel& timing_override) {
  if (std::find(ranks_list.begin(), ranks_list.end(), 1) == ranks_list.end())
    throw std::invalid_argument("run_scaling_sweep: threads list must include 1");
  if (!timing_override)
    for (const int P : ranks_list)
      if (P != 1)
        throw std::invalid_argument(
            "run_scaling_sweep: measuring P > 1 needs one process per GPU "
            "(bench.py --gpus P); pass a timing model for P > 1");
  SweepResult out;
  for (const auto& dims : dims_list) {
    std::vector<BenchRecord> group;
    for (const int P : ranks_list) {
      BenchRecord rec;
      if (timing_override) {
        rec.bp = bp_name(bp);
        rec.p = p;
        rec.q = bp_quadrature_points(bp, p);
        rec.E = int64_t(dims[0]) * dims[1] * dims[2];
        rec.n = bp_dof_count(bp, p, dims);
        rec.P = P;
        rec.iterations = iterations;
        rec.seconds = timing_override(rec.n, P);
        rec.dofs_rate = double(rec.n) * rec.iterations / rec.seconds;
        rec.n_per_rank = double(rec.n) / rec.P;
      } else {
        BpConfig c;
        c.bp = bp;
        c.p = p;
        c.dims = dims;
        c.deformation = deformation;
        c.fixed_iterations = iterations;
        rec = run_bench(c);
      }
      group.push_back(rec);
    }
    double t1 = 0;
    for (const auto& r : group)
      if (r.P == 1) t1 = r.seconds;
    for (auto& r : group) {
      ScalingRow row;
      row.T_1 = t1;
      row.T_P = r.seconds;
      row.eta = t1 / (r.P * r.seconds);
      row.record = std::move(r);
      out.rows.push_back(std::move(row));
    }
  }
  out.summary = scaling_summary(out.rows);
  return out;
}

ScalingSummary scaling_summary(std::vector<ScalingRow>& rows) {
  std::sort(rows.begin(), rows.end(), [](const ScalingRow& a, const ScalingRow& b) {
    if (a.record.n_per_rank != b.record.n_per_rank) return a.record.n_per_rank < b.record.n_per_rank;
    if (a.record.n != b.record.n) return a.record.n < b.record.n;
    return a.record.P < b.record.P;
  });
  ScalingSummary s;
  for (const auto& r : rows) s.r_max = std::max(s.r_max, r.record.dofs_rate / r.record.P);
  // first upward crossing of eta = 0.8 among the P > 1 rows (P = 1 has eta 1)
  const ScalingRow* prev = nullptr;
  for (const auto& r : rows) {
    if (r.record.P <= 1) continue;
    if (prev && prev->eta < 0.8 && r.eta >= 0.8) {
      const double x0 = std::log(prev->record.n_per_rank), x1 = std::log(r.record.n_per_rank);
      const double t = (0.8 - prev->eta) / (r.eta - prev->eta);
      s.n08_per_rank = std::exp(x0 + t * (x1 - x0));
      break;
    }
    prev = &r;
  }
  double num = 0, den = 0;
  if (s.r_max > 0)
    for (const auto& r : rows) {
      const double xi = double(r.record.n) / (r.eta * r.record.P * s.r_max);
      num += r.T_P * xi;
      den += xi * xi;
    }
  s.work_constant = den > 0 ? num / den : 0.0;
  return s;
}

double time_to_solution(double work_constant, double n, double eta, double P, double r_max) {
  return work_constant * n / (eta * P * r_max);
}

std::string format_double(double v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v);
  return std::string(buf, res.ptr);
}

namespace {
std::string json_double(double v) {  // JSON number, round-trip exact
  if (!std::isfinite(v)) return "null";
  std::string s = format_double(v);
  if (s.find_first_of(".eE") == std::string::npos) s += ".0";
  return s;
}
std::string json_string(const std::string& v) {
  std::string o = "\"";
  for (const char c : v) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}
std::string csv_field(const std::string& v) {
  if (v.find_first_of(",\"\r\n") == std::string::npos) return v;
  std::string o = "\"";
  for (const char c : v) o += (c == '"') ? std::string("\"\"") : std::string(1, c);
  return o + "\"";
}
}  // namespace

std::string bench_record_json(const BenchRecord& r) {
  return "{\"bp\":" + json_string(r.bp) + ",\"p\":" + std::to_string(r.p) +
         ",\"q\":" + std::to_string(r.q) + ",\"E\":" + std::to_string(r.E) +
         ",\"n\":" + std::to_string(r.n) + ",\"P\":" + std::to_string(r.P) +
         ",\"iterations\":" + std::to_string(r.iterations) + ",\"seconds\":" +
         json_double(r.seconds) + ",\"dofs_rate\":" + json_double(r.dofs_rate) +
         ",\"n_per_rank\":" + json_double(r.n_per_rank) + "}";
}

std::string sweep_csv_header() { return "bp,p,q,E,n,P,iters,seconds,dofs_rate,n_per_rank,eta"; }

std::string sweep_csv(const SweepResult& result) {
  std::string o = sweep_csv_header() + "\n";
  for (const auto& row : result.rows) {
    const BenchRecord& r = row.record;
    o += csv_field(r.bp) + "," + std::to_string(r.p) + "," + std::to_string(r.q) + "," +
         std::to_string(r.E) + "," + std::to_string(r.n) + "," + std::to_string(r.P) + "," +
         std::to_string(r.iterations) + "," + format_double(r.seconds) + "," +
         format_double(r.dofs_rate) + "," + format_double(r.n_per_rank) + "," +
         format_double(row.eta) + "\n";
  }
  return o;
}

std::vector<double> assemble_dense(BpProblem& problem) {
  const int64_t n = problem.size();
  if (n > 20000)
    throw std::invalid_argument("reference_assemble: problem too large (m*n_L = " +
                                std::to_string(n) + " > 20000)");
  std::vector<double> A(size_t(n) * n), e(size_t(n), 0.0), col(static_cast<size_t>(n));
  DeviceBuffer de(problem.device, size_t(n)), dy(problem.device, size_t(n));
  for (int64_t j = 0; j < n; ++j) {
    e[size_t(j)] = 1.0;
    de.upload(e.data(), e.size());
    e[size_t(j)] = 0.0;
    problem.op->apply_device(de.data(), dy.data());
    dy.download(col.data(), col.size());
    for (int64_t i = 0; i < n; ++i) A[size_t(i * n + j)] = col[size_t(i)];
  }
  return A;
}

}  // namespace hexfem_b200
