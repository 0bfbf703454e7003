// Partitioned-box support: communicators, the interface
// sum-exchange and the owner-weighted all-reduce that let one structured
// sub-box per GPU run the same fused PCG as the single-domain path.
//
// The reference has no distributed layer (threads over one address space,
// proj/src/parallel.cpp:17-67); its paper's codes use MPI + gslib
// gather-scatter for the assembly P operator.
// Here the exchange is dimension ordered — x planes, then y, then z — so an
// edge or corner node shared by 4 or 8 sub-boxes is summed through its face
// neighbours without diagonal messages.  Every copy of a shared node ends
// with the same bits: each phase adds two already-equal partial sums, and
// floating-point addition commutes.
//
// Backends:
//   NcclComm   libnccl.so.2 opened with dlopen (torch's copy when torch
//              already loaded one): grouped ncclSend/ncclRecv per axis and
//              an in-place ncclAllReduce(f64, sum).  Stream ordered and CUDA
//              graph capturable.
//   GroupComm  N sub-domains in one process, one host thread each (tests on
//              a single GPU).  Host-synchronous: stream sync + barrier around
//              every exchange, rank-ordered host sums for all-reduce.
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

#include "../../include/hxf.h"
#include "capi_internal.h"

namespace hxf {

struct Xfer {
  int peer;
  const double* send;
  double* recv;
  size_t n;
};

struct Comm {
  int rank = 0, size = 1;
  bool graph_safe = false;  // may be captured into a CUDA graph
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* dev, size_t n, cudaStream_t s) = 0;
  // every rank posts its transfers; a transfer to `peer` pairs with that
  // peer's transfer back, in posting order
  virtual void exchange(const std::vector<Xfer>& xs, cudaStream_t s) = 0;
};

namespace {

// ---- NCCL through dlopen ---------------------------------------------------
struct NcclId {
  char internal[HXF_COMM_ID_BYTES];
};
using ncclComm_t = void*;
constexpr int kNcclFloat64 = 8;  // ncclDataType_t::ncclFloat64
constexpr int kNcclSum = 0;      // ncclRedOp_t::ncclSum

struct NcclApi {
  int (*get_unique_id)(NcclId*) = nullptr;
  int (*comm_init_rank)(ncclComm_t*, int, NcclId, int) = nullptr;
  int (*comm_destroy)(ncclComm_t) = nullptr;
  int (*comm_count)(ncclComm_t, int*) = nullptr;
  int (*comm_user_rank)(ncclComm_t, int*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  const char* (*error_string)(int) = nullptr;
  std::string load_error;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // prefer a libnccl already in the process (torch's), else the loader's
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW);
    if (!h) {
      const char* e = dlerror();
      a.load_error = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
      return a;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn && a.load_error.empty()) a.load_error = std::string("libnccl lacks ") + name;
    };
    sym(a.get_unique_id, "ncclGetUniqueId");
    sym(a.comm_init_rank, "ncclCommInitRank");
    sym(a.comm_destroy, "ncclCommDestroy");
    sym(a.comm_count, "ncclCommCount");
    sym(a.comm_user_rank, "ncclCommUserRank");
    sym(a.all_reduce, "ncclAllReduce");
    sym(a.send, "ncclSend");
    sym(a.recv, "ncclRecv");
    sym(a.group_start, "ncclGroupStart");
    sym(a.group_end, "ncclGroupEnd");
    sym(a.error_string, "ncclGetErrorString");
    return a;
  }();
  if (!api.load_error.empty()) fail(HXF_ENCCL, api.load_error);
  return api;
}

void nck(int r, const char* what) {
  if (r != 0) {
    const NcclApi& a = nccl();
    fail(HXF_ENCCL, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "error"));
  }
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  bool owned = true;
  ~NcclComm() override {
    if (comm && owned) nccl().comm_destroy(comm);
  }
  void allreduce_sum(double* dev, size_t n, cudaStream_t s) override {
    nck(nccl().all_reduce(dev, dev, n, kNcclFloat64, kNcclSum, comm, s), "ncclAllReduce");
  }
  void exchange(const std::vector<Xfer>& xs, cudaStream_t s) override {
    const NcclApi& a = nccl();
    nck(a.group_start(), "ncclGroupStart");
    for (const Xfer& x : xs) {
      nck(a.send(x.send, x.n, kNcclFloat64, x.peer, comm, s), "ncclSend");
      nck(a.recv(x.recv, x.n, kNcclFloat64, x.peer, comm, s), "ncclRecv");
    }
    nck(a.group_end(), "ncclGroupEnd");
  }
};

// ---- in-process group --------------------------------------------------------
struct GroupShared {
  int size = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<std::vector<double>> vals;  // all-reduce staging, per rank
  std::vector<std::vector<Xfer>> posted;  // exchange posts, per rank

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const int64_t gen = generation;
    if (++arrived == size) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; }))
      fail(HXF_ENCCL, "hxf group comm: barrier timed out (a rank stopped calling collectives)");
  }
};

struct GroupComm final : Comm {
  std::shared_ptr<GroupShared> g;
  void allreduce_sum(double* dev, size_t n, cudaStream_t s) override {
    std::vector<double>& mine = g->vals[size_t(rank)];
    mine.resize(n);
    ck(cudaMemcpyAsync(mine.data(), dev, n * 8, cudaMemcpyDeviceToHost, s), "group allreduce");
    ck(cudaStreamSynchronize(s), "group allreduce");
    g->barrier();
    std::vector<double> sum(n, 0.0);
    for (int r = 0; r < size; ++r) {  // rank order: identical bits on every rank
      if (g->vals[size_t(r)].size() != n) fail(HXF_ENCCL, "group allreduce: length mismatch");
      for (size_t i = 0; i < n; ++i) sum[i] += g->vals[size_t(r)][i];
    }
    g->barrier();
    ck(cudaMemcpyAsync(dev, sum.data(), n * 8, cudaMemcpyHostToDevice, s), "group allreduce");
    ck(cudaStreamSynchronize(s), "group allreduce");
  }
  void exchange(const std::vector<Xfer>& xs, cudaStream_t s) override {
    ck(cudaStreamSynchronize(s), "group exchange");  // packed planes complete
    g->posted[size_t(rank)] = xs;
    g->barrier();
    std::vector<int> used(size_t(size), 0);
    for (const Xfer& x : xs) {
      if (x.peer < 0 || x.peer >= size) fail(HXF_EINVAL, "group exchange: bad peer");
      const Xfer* match = nullptr;
      int seen = 0;
      for (const Xfer& y : g->posted[size_t(x.peer)])
        if (y.peer == rank && seen++ == used[size_t(x.peer)]) {
          match = &y;
          break;
        }
      ++used[size_t(x.peer)];
      if (!match || match->n != x.n) fail(HXF_ENCCL, "group exchange: unmatched transfer");
      ck(cudaMemcpyAsync(x.recv, match->send, x.n * 8, cudaMemcpyDefault, s), "group exchange");
    }
    ck(cudaStreamSynchronize(s), "group exchange");
    g->barrier();  // peers' send planes may be reused from here on
  }
};

// ---- peer-to-peer (NVLink / same-device) mailboxes ---------------------------
// Every rank owns one device allocation (exported by CUDA IPC between
// processes, or shared directly inside one process):
//   mail  [2][N][cap] f64   exchange slots, by parity and source rank
//   ar    [2][N][8]   f64   all-reduce slots
//   xflag [2][N]      u64   exchange arrival counters (+1 per put CTA)
//   aflag [2][N]      u64   all-reduce arrival values
//   state: sseq[N], rseq[N], sdone[N], rdone[N], aseq (u64, local only)
// A put kernel stores a packed plane straight into the PEER's slot (remote
// stores over NVLink; plain stores on one device), fences at system scope
// and bumps the peer's counter; the matching get kernel spins on its own
// counter and copies the slot out.  Sequence numbers live on the device, so
// the kernels are CUDA-graph capturable, and every slot is double-buffered by
// the pair's transfer parity: a put of transfer k+2 can only run after its
// rank's get of k+1, which the peer posted after reading transfer k.
constexpr int kP2pMax = 16;
constexpr int kP2pBlocks = 32;

struct P2pLayout {
  int N;
  int64_t cap;
  __host__ __device__ size_t mail_off() const { return 0; }
  __host__ __device__ size_t ar_off() const { return size_t(2) * N * size_t(cap) * 8; }
  __host__ __device__ size_t xflag_off() const { return ar_off() + size_t(2) * N * 8 * 8; }
  __host__ __device__ size_t aflag_off() const { return xflag_off() + size_t(2) * N * 8; }
  __host__ __device__ size_t state_off() const { return aflag_off() + size_t(2) * N * 8; }
  __host__ __device__ size_t bytes() const { return state_off() + size_t(4 * N + 1) * 8; }
};

struct P2pPeers {
  char* base[kP2pMax];
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// spin (bounded: a lost peer traps instead of hanging the GPU)
__device__ __forceinline__ void wait_at_least(const unsigned long long* p, unsigned long long v) {
  long long spins = 0;
  while (ld_acquire_sys(p) < v) {
    __nanosleep(64);
    if (++spins > (1ll << 26)) __trap();
  }
}

__global__ void p2p_put_kernel(P2pPeers pe, P2pLayout L, int rank, int peer, const double* __restrict__ send,
                               int64_t n) {
  char* mine = pe.base[rank];
  unsigned long long* st = reinterpret_cast<unsigned long long*>(mine + L.state_off());
  const unsigned long long k = st[peer];  // sseq[peer]: updated only by the last CTA
  const int par = int(k & 1);
  double* dst = reinterpret_cast<double*>(pe.base[peer] + L.mail_off()) +
                (size_t(par) * L.N + rank) * size_t(L.cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = send[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    unsigned long long* flag = reinterpret_cast<unsigned long long*>(pe.base[peer] + L.xflag_off()) +
                               par * L.N + rank;
    atomicAdd_system(flag, 1ull);
    if (atomicAdd(&st[2 * L.N + peer], 1ull) == gridDim.x - 1) {  // sdone: last CTA
      st[2 * L.N + peer] = 0;
      st[peer] = k + 1;
    }
  }
}

__global__ void p2p_get_kernel(P2pPeers pe, P2pLayout L, int rank, int peer, double* __restrict__ recv,
                               int64_t n) {
  char* mine = pe.base[rank];
  unsigned long long* st = reinterpret_cast<unsigned long long*>(mine + L.state_off());
  const unsigned long long j = st[L.N + peer];  // rseq[peer]
  const int par = int(j & 1);
  const unsigned long long* flag =
      reinterpret_cast<const unsigned long long*>(mine + L.xflag_off()) + par * L.N + peer;
  const unsigned long long target = (unsigned long long)kP2pBlocks * ((j >> 1) + 1);
  if (threadIdx.x == 0) wait_at_least(flag, target);
  __syncthreads();
  (void)ld_acquire_sys(flag);  // every thread acquires the peer's stores
  const double* src = reinterpret_cast<const double*>(mine + L.mail_off()) +
                      (size_t(par) * L.N + peer) * size_t(L.cap);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    recv[i] = src[i];
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&st[3 * L.N + peer], 1ull) == gridDim.x - 1) {  // rdone
    st[3 * L.N + peer] = 0;
    st[L.N + peer] = j + 1;
  }
}

// one CTA: put this rank's n (<= 8) values into every rank's slot, wait for
// all N, sum in rank order (identical bits on every rank)
__global__ void p2p_allreduce_kernel(P2pPeers pe, P2pLayout L, int rank, double* v, int n) {
  char* mine = pe.base[rank];
  unsigned long long* st = reinterpret_cast<unsigned long long*>(mine + L.state_off());
  const unsigned long long a = st[4 * L.N];
  const int par = int(a & 1);
  const unsigned long long val = (a >> 1) + 1;
  const int t = threadIdx.x;
  for (int i = t; i < L.N * n; i += blockDim.x) {
    const int q = i / n, c = i - q * n;
    reinterpret_cast<double*>(pe.base[q] + L.ar_off())[(size_t(par) * L.N + rank) * 8 + c] = v[c];
  }
  __syncthreads();
  if (t == 0) {
    __threadfence_system();
    for (int q = 0; q < L.N; ++q)
      atomicExch_system(reinterpret_cast<unsigned long long*>(pe.base[q] + L.aflag_off()) + par * L.N + rank,
                        val);
    const unsigned long long* fl = reinterpret_cast<const unsigned long long*>(mine + L.aflag_off()) + par * L.N;
    for (int q = 0; q < L.N; ++q) wait_at_least(fl + q, val);
  }
  __syncthreads();
  (void)ld_acquire_sys(reinterpret_cast<const unsigned long long*>(mine + L.aflag_off()) + par * L.N);
  if (t < n) {
    const double* slots = reinterpret_cast<const double*>(mine + L.ar_off()) + size_t(par) * L.N * 8;
    double s = 0.0;
    for (int q = 0; q < L.N; ++q) s += slots[q * 8 + t];
    v[t] = s;
  }
  __syncthreads();
  if (t == 0) st[4 * L.N] = a + 1;
}

struct P2pComm final : Comm {
  P2pLayout L{};
  P2pPeers pe{};
  void* local = nullptr;       // this rank's allocation (owned when allocated here)
  bool owns_local = false;
  std::vector<void*> opened;   // IPC-opened peer allocations
  ~P2pComm() override {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    if (owns_local && local) cudaFree(local);
  }
  void allreduce_sum(double* dev, size_t n, cudaStream_t s) override {
    for (size_t off = 0; off < n; off += 8) {
      const int k = int(std::min<size_t>(8, n - off));
      p2p_allreduce_kernel<<<1, 64, 0, s>>>(pe, L, rank, dev + off, k);
      count_launch(1);
      ck(cudaGetLastError(), "p2p allreduce");
    }
  }
  void exchange(const std::vector<Xfer>& xs, cudaStream_t s) override {
    for (const Xfer& x : xs) {
      if (x.peer < 0 || x.peer >= size || x.peer == rank) fail(HXF_EINVAL, "p2p exchange: bad peer");
      if (int64_t(x.n) > L.cap) fail(HXF_EINVAL, "p2p exchange: plane larger than the mailbox");
      p2p_put_kernel<<<kP2pBlocks, 256, 0, s>>>(pe, L, rank, x.peer, x.send, int64_t(x.n));
      count_launch(1);
      ck(cudaGetLastError(), "p2p put");
    }
    for (const Xfer& x : xs) {
      p2p_get_kernel<<<kP2pBlocks, 256, 0, s>>>(pe, L, rank, x.peer, x.recv, int64_t(x.n));
      count_launch(1);
      ck(cudaGetLastError(), "p2p get");
    }
  }
};

// ---- plane kernels -----------------------------------------------------------
struct Plane {
  int axis;
  int64_t fixed, nu, nv, NX, NY, n_L, count;  // count = nu * nv
};

__device__ __forceinline__ int64_t plane_node(const Plane& P, int64_t t) {
  const int64_t u = t % P.nu, v = t / P.nu;
  const int64_t ix = P.axis == 0 ? P.fixed : u;
  const int64_t iy = P.axis == 1 ? P.fixed : (P.axis == 0 ? u : v);
  const int64_t iz = P.axis == 2 ? P.fixed : v;
  return ix + P.NX * (iy + P.NY * iz);
}

__global__ void plane_pack_kernel(Plane P, int m, const double* __restrict__ v,
                                  double* __restrict__ buf) {
  const int64_t total = P.count * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / P.count, t = i - c * P.count;
    buf[i] = v[c * P.n_L + plane_node(P, t)];
  }
}

__global__ void plane_add_kernel(Plane P, int m, double* __restrict__ v,
                                 const double* __restrict__ buf) {
  const int64_t total = P.count * m;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i / P.count, t = i - c * P.count;
    v[c * P.n_L + plane_node(P, t)] += buf[i];
  }
}

// constrained rows: owner keeps `value`, other copies 0 (a following
// sum-exchange then leaves exactly `value` everywhere)
__global__ void set_constrained_kernel(int64_t n_L, int m, const uint32_t* __restrict__ mask,
                                       const uint32_t* __restrict__ own, double value,
                                       double* __restrict__ v) {
  for (int64_t node = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; node < n_L;
       node += (int64_t)gridDim.x * blockDim.x) {
    if (!((mask[node >> 5] >> (node & 31)) & 1u)) continue;
    const bool owned = !own || ((own[node >> 5] >> (node & 31)) & 1u);
    for (int c = 0; c < m; ++c) v[c * n_L + node] = owned ? value : 0.0;
  }
}

int grid_for(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return int(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(num_sms()) * 8)));
}

Plane make_plane(const hxf_op* op, int axis, int side) {
  Plane P{};
  P.axis = axis;
  const int64_t N[3] = {op->NX, op->NY, op->NZ};
  P.fixed = side ? N[axis] - 1 : 0;
  P.nu = axis == 0 ? op->NY : op->NX;
  P.nv = axis == 2 ? op->NY : op->NZ;
  P.NX = op->NX;
  P.NY = op->NY;
  P.n_L = op->n_L;
  P.count = P.nu * P.nv;
  return P;
}

}  // namespace

bool op_partitioned(const hxf_op* op) { return op && op->comm; }
bool op_graph_safe(const hxf_op* op) { return !op->comm || op->comm->graph_safe; }

void op_allreduce(hxf_op* op, double* dev, int n, cudaStream_t s) {
  if (op->comm) op->comm->allreduce_sum(dev, size_t(n), s);
}

void op_halo_sum(hxf_op* op, double* v, cudaStream_t s) {
  if (!op->comm) return;
  const int m = op->m;
  const int64_t maxplane = std::max({op->NY * op->NZ, op->NX * op->NZ, op->NX * op->NY}) * m;
  double* buf = op->w_halo.ensure(size_t(4 * maxplane));
  for (int axis = 0; axis < 3; ++axis) {
    std::vector<Xfer> xs;
    Plane planes[2];
    for (int side = 0; side < 2; ++side) {
      const int peer = op->neighbor[axis][side];
      if (peer < 0) continue;
      planes[side] = make_plane(op, axis, side);
      const size_t n = size_t(planes[side].count) * m;
      double* send = buf + size_t(side) * maxplane;
      double* recv = buf + size_t(2 + side) * maxplane;
      plane_pack_kernel<<<grid_for(int64_t(n)), 256, 0, s>>>(planes[side], m, v, send);
      count_launch(1);
      ck(cudaGetLastError(), "halo pack");
      xs.push_back({peer, send, recv, n});
    }
    if (xs.empty()) continue;
    op->comm->exchange(xs, s);
    for (int side = 0; side < 2; ++side) {
      if (op->neighbor[axis][side] < 0) continue;
      const size_t n = size_t(planes[side].count) * m;
      plane_add_kernel<<<grid_for(int64_t(n)), 256, 0, s>>>(planes[side], m, v,
                                                            buf + size_t(2 + side) * maxplane);
      count_launch(1);
      ck(cudaGetLastError(), "halo add");
    }
  }
}

void op_set_constrained(hxf_op* op, double* v, double value, cudaStream_t s) {
  if (!op->d_mask) return;
  set_constrained_kernel<<<grid_for(op->n_L), 256, 0, s>>>(op->n_L, op->m, op->d_mask, op->d_own,
                                                           value, v);
  count_launch(1);
  ck(cudaGetLastError(), "set constrained");
}

}  // namespace hxf

struct hxf_comm {
  std::unique_ptr<hxf::Comm> impl;
  hxf_ctx* ctx = nullptr;
};
struct hxf_comm_group {
  std::shared_ptr<hxf::GroupShared> shared;
};

namespace {
template <class F>
int guarded_dist(F&& f) {
  try {
    f();
    return HXF_OK;
  } catch (const HxfError& e) {
    hxf::set_last_error(e.msg.c_str());
    return e.code;
  } catch (const std::exception& e) {
    hxf::set_last_error(e.what());
    return HXF_ECUDA;
  }
}
}  // namespace

extern "C" {

int hxf_comm_unique_id(unsigned char id[HXF_COMM_ID_BYTES]) {
  return guarded_dist([&] {
    if (!id) fail(HXF_EINVAL, "hxf_comm_unique_id: NULL");
    NcclId nid{};
    nck(nccl().get_unique_id(&nid), "ncclGetUniqueId");
    std::memcpy(id, nid.internal, HXF_COMM_ID_BYTES);
  });
}

int hxf_comm_create_nccl(hxf_ctx* ctx, int nranks, int rank, const unsigned char id[HXF_COMM_ID_BYTES],
                         hxf_comm** out) {
  return guarded_dist([&] {
    if (!ctx || !id || !out) fail(HXF_EINVAL, "hxf_comm_create_nccl: NULL argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(HXF_EINVAL, "hxf_comm_create_nccl: bad rank");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    NcclId nid{};
    std::memcpy(nid.internal, id, HXF_COMM_ID_BYTES);
    auto c = std::make_unique<NcclComm>();
    nck(nccl().comm_init_rank(&c->comm, nranks, nid, rank), "ncclCommInitRank");
    c->rank = rank;
    c->size = nranks;
    c->graph_safe = true;
    auto* h = new hxf_comm();
    h->impl = std::move(c);
    h->ctx = ctx;
    *out = h;
  });
}

int hxf_comm_wrap_nccl(hxf_ctx* ctx, void* nccl_comm, hxf_comm** out) {
  return guarded_dist([&] {
    if (!ctx || !nccl_comm || !out) fail(HXF_EINVAL, "hxf_comm_wrap_nccl: NULL argument");
    auto c = std::make_unique<NcclComm>();
    c->comm = nccl_comm;
    c->owned = false;
    nck(nccl().comm_count(nccl_comm, &c->size), "ncclCommCount");
    nck(nccl().comm_user_rank(nccl_comm, &c->rank), "ncclCommUserRank");
    c->graph_safe = true;
    auto* h = new hxf_comm();
    h->impl = std::move(c);
    h->ctx = ctx;
    *out = h;
  });
}

int hxf_comm_group_create(int nranks, hxf_comm_group** out) {
  return guarded_dist([&] {
    if (!out || nranks < 1) fail(HXF_EINVAL, "hxf_comm_group_create: bad argument");
    auto* g = new hxf_comm_group();
    g->shared = std::make_shared<GroupShared>();
    g->shared->size = nranks;
    g->shared->vals.resize(size_t(nranks));
    g->shared->posted.resize(size_t(nranks));
    *out = g;
  });
}

int hxf_comm_group_destroy(hxf_comm_group* group) {
  delete group;
  return HXF_OK;
}

int hxf_comm_create_group(hxf_ctx* ctx, hxf_comm_group* group, int rank, hxf_comm** out) {
  return guarded_dist([&] {
    if (!ctx || !group || !out) fail(HXF_EINVAL, "hxf_comm_create_group: NULL argument");
    if (rank < 0 || rank >= group->shared->size) fail(HXF_EINVAL, "hxf_comm_create_group: bad rank");
    auto c = std::make_unique<GroupComm>();
    c->g = group->shared;
    c->rank = rank;
    c->size = group->shared->size;
    c->graph_safe = false;
    auto* h = new hxf_comm();
    h->impl = std::move(c);
    h->ctx = ctx;
    *out = h;
  });
}

int hxf_comm_p2p_alloc(hxf_ctx* ctx, int nranks, int64_t cap, void** base,
                       unsigned char handle[HXF_COMM_IPC_HANDLE_BYTES]) {
  return guarded_dist([&] {
    if (!ctx || !base) fail(HXF_EINVAL, "hxf_comm_p2p_alloc: NULL argument");
    if (nranks < 1 || nranks > kP2pMax || cap < 1) fail(HXF_EINVAL, "hxf_comm_p2p_alloc: bad size");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    const P2pLayout L{nranks, cap};
    void* p = nullptr;
    ck(cudaMalloc(&p, L.bytes()), "p2p mailbox");
    ck(cudaMemset(p, 0, L.bytes()), "p2p mailbox");
    ck(cudaDeviceSynchronize(), "p2p mailbox");
    if (handle) {
      cudaIpcMemHandle_t h{};
      ck(cudaIpcGetMemHandle(&h, p), "cudaIpcGetMemHandle");
      std::memcpy(handle, &h, sizeof h);
    }
    *base = p;
  });
}

int hxf_comm_create_p2p(hxf_ctx* ctx, int nranks, int rank, int64_t cap, void* const* bases,
                        const unsigned char* handles, hxf_comm** out) {
  return guarded_dist([&] {
    if (!ctx || !out || (!bases && !handles)) fail(HXF_EINVAL, "hxf_comm_create_p2p: NULL argument");
    if (nranks < 1 || nranks > kP2pMax || rank < 0 || rank >= nranks || cap < 1)
      fail(HXF_EINVAL, "hxf_comm_create_p2p: bad rank / size");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    auto c = std::make_unique<P2pComm>();
    c->L = P2pLayout{nranks, cap};
    c->rank = rank;
    c->size = nranks;
    c->graph_safe = true;
    for (int q = 0; q < nranks; ++q) {
      if (bases && bases[q]) {  // same process: direct pointers
        c->pe.base[q] = static_cast<char*>(bases[q]);
        continue;
      }
      if (!handles) fail(HXF_EINVAL, "hxf_comm_create_p2p: rank without a mailbox");
      cudaIpcMemHandle_t h{};
      std::memcpy(&h, handles + size_t(q) * HXF_COMM_IPC_HANDLE_BYTES, sizeof h);
      void* p = nullptr;
      ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
      c->opened.push_back(p);
      c->pe.base[q] = static_cast<char*>(p);
    }
    if (!c->pe.base[rank]) fail(HXF_EINVAL, "hxf_comm_create_p2p: own mailbox missing");
    auto* h = new hxf_comm();
    h->impl = std::move(c);
    h->ctx = ctx;
    *out = h;
  });
}

int hxf_comm_p2p_free(hxf_ctx* ctx, void* base) {
  return guarded_dist([&] {
    if (!ctx) fail(HXF_EINVAL, "hxf_comm_p2p_free: NULL context");
    if (base) {
      ck(cudaDeviceSynchronize(), "p2p mailbox");
      ck(cudaFree(base), "p2p mailbox");
    }
  });
}

int hxf_comm_destroy(hxf_comm* comm) {
  return guarded_dist([&] {
    if (!comm) return;
    if (comm->ctx) cudaStreamSynchronize(comm->ctx->stream);
    delete comm;
  });
}

int hxf_comm_rank(const hxf_comm* comm) { return comm ? comm->impl->rank : -1; }
int hxf_comm_size(const hxf_comm* comm) { return comm ? comm->impl->size : 0; }

int hxf_comm_allreduce_sum(hxf_comm* comm, double* dev, int64_t n, void* stream) {
  return guarded_dist([&] {
    if (!comm || (!dev && n > 0) || n < 0) fail(HXF_EINVAL, "hxf_comm_allreduce_sum: bad argument");
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : comm->ctx->stream;
    if (n > 0) comm->impl->allreduce_sum(dev, size_t(n), s);
  });
}

int hxf_operator_set_partition(hxf_op* op, hxf_comm* comm, const hxf_partition_desc* desc) {
  return guarded_dist([&] {
    if (!op || !comm || !desc) fail(HXF_EINVAL, "hxf_operator_set_partition: NULL argument");
    if (!op->structured)
      fail(HXF_EUNSUPPORTED, "hxf_operator_set_partition: needs a structured-box operator");
    for (int a = 0; a < 3; ++a)
      for (int s = 0; s < 2; ++s) {
        const int nb = desc->neighbor[a][s];
        if (nb < -1 || nb >= comm->impl->size || nb == comm->impl->rank)
          fail(HXF_EINVAL, "hxf_operator_set_partition: bad neighbour rank");
      }
    const int64_t NX = op->NX, NY = op->NY, NZ = op->NZ;
    // owner: not on a low face plane shared with a neighbour (exactly one
    // copy of every interface node satisfies this)
    std::vector<uint32_t> own(size_t((op->n_L + 31) / 32), 0u);
    const bool lx = desc->neighbor[0][0] >= 0, ly = desc->neighbor[1][0] >= 0,
               lz = desc->neighbor[2][0] >= 0;
    int64_t node = 0;
    for (int64_t iz = 0; iz < NZ; ++iz)
      for (int64_t iy = 0; iy < NY; ++iy)
        for (int64_t ix = 0; ix < NX; ++ix, ++node)
          if (!((lx && ix == 0) || (ly && iy == 0) || (lz && iz == 0)))
            own[size_t(node >> 5)] |= 1u << (node & 31);
    if (!op->d_own) op->d_own = dalloc<uint32_t>(own.size());
    ck(cudaMemcpy(op->d_own, own.data(), own.size() * 4, cudaMemcpyHostToDevice), "owner upload");
    // boundary-first element order: elements with a face on an interface
    // plane (the only writers of shared nodes), then the interior
    std::vector<int> bnd, inr;
    const int nx = op->nx, ny = op->ny, nz = op->nz;
    const int(*nb)[2] = desc->neighbor;
    for (int ez = 0; ez < nz; ++ez)
      for (int ey = 0; ey < ny; ++ey)
        for (int ex = 0; ex < nx; ++ex) {
          const bool b = (ex == 0 && nb[0][0] >= 0) || (ex == nx - 1 && nb[0][1] >= 0) ||
                         (ey == 0 && nb[1][0] >= 0) || (ey == ny - 1 && nb[1][1] >= 0) ||
                         (ez == 0 && nb[2][0] >= 0) || (ez == nz - 1 && nb[2][1] >= 0);
          (b ? bnd : inr).push_back(ex + nx * (ey + ny * ez));
        }
    if (op->d_elist) cudaFree(op->d_elist);
    op->d_elist = dalloc<int>(size_t(op->E));
    ck(cudaMemcpy(op->d_elist, bnd.data(), bnd.size() * 4, cudaMemcpyHostToDevice), "elist");
    ck(cudaMemcpy(op->d_elist + bnd.size(), inr.data(), inr.size() * 4, cudaMemcpyHostToDevice),
       "elist");
    op->n_bnd = int64_t(bnd.size());
    op->n_int = int64_t(inr.size());
    if (!op->s_comm) {
      int lo = 0, hi = 0;
      ck(cudaDeviceGetStreamPriorityRange(&lo, &hi), "priority");
      // highest priority: the exchange's kernels are scheduled ahead of the
      // interior elements' CTAs as SM slots free up
      ck(cudaStreamCreateWithPriority(&op->s_comm, cudaStreamNonBlocking, hi), "comm stream");
      ck(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming), "event");
    }
    op->comm = comm->impl.get();
    std::memcpy(op->neighbor, desc->neighbor, sizeof op->neighbor);
    op->drop_graphs();
  });
}

int hxf_operator_halo_sum(hxf_op* op, double* v, hxf_memspace space) {
  return guarded_dist([&] {
    if (!op || !v) fail(HXF_EINVAL, "hxf_operator_halo_sum: NULL argument");
    cudaStream_t s = op->ctx->stream;
    const size_t n = size_t(op->m) * size_t(op->n_L);
    double* dv = v;
    if (space == HXF_HOST) {
      dv = op->ctx->scratch_a.ensure(n);
      ck(cudaMemcpyAsync(dv, v, n * 8, cudaMemcpyHostToDevice, s), "halo H2D");
    }
    op_halo_sum(op, dv, s);
    if (space == HXF_HOST)
      ck(cudaMemcpyAsync(v, dv, n * 8, cudaMemcpyDeviceToHost, s), "halo D2H");
    ck(cudaStreamSynchronize(s), "halo sum");
  });
}

}  // extern "C"
