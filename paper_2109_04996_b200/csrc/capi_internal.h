// Internal host-side definitions shared by the C-ABI translation units
// (capi.cu, dist.cu): error helpers, device allocation, and the context /
// operator handle structs behind the opaque hxf_ctx / hxf_op.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "aux_kernels.h"
#include "hxf_internal.h"
#include "pcg_kernels.h"

namespace hxf {
struct Comm;  // dist.cu
}

namespace hxf_detail {
struct HxfError {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw HxfError{code, msg}; }

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(HXF_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* dalloc(size_t n) {
  void* p = nullptr;
  ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
  return static_cast<T*>(p);
}

inline void h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpy H2D");
}
inline void d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "cudaMemcpy D2H");
}

struct DevVec {
  double* p = nullptr;
  size_t n = 0;
  double* ensure(size_t want) {
    if (want > n) {
      if (p) cudaFree(p);
      p = dalloc<double>(want);
      n = want;
    }
    return p;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace hxf_detail

using namespace hxf;
using namespace hxf_detail;

struct hxf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  void* nccl = nullptr;
  DevVec scratch_a, scratch_b, scratch_c, scratch_d;  // API-surface staging
};

struct hxf_op {
  hxf_ctx* ctx = nullptr;
  int p = 0, q = 0, m = 1, P = 0, Q = 0;
  int64_t E = 0, n_L = 0;
  bool interp = false;
  bool symmetric = false;  // centro-symmetric 1-D matrices (even-odd kernels usable)
  std::vector<double> B, Dq;  // kernel-parameter matrices
  double alpha = 0, beta = 0;
  bool structured = false;
  int nx = 0, ny = 0, nz = 0;
  int64_t NX = 0, NY = 0, NZ = 0;
  int* d_idx = nullptr;
  int cons_mode = 0;
  int bnd_faces = 0;
  uint32_t* d_mask = nullptr;
  int64_t ncons = 0;
  double* d_qd_diff = nullptr;
  int64_t diff_stride = 0;
  double* d_qd_mass = nullptr;
  int64_t mass_stride = 0;
  double* d_part = nullptr;
  double *d_B = nullptr, *d_G = nullptr, *d_Bt = nullptr, *d_Gt = nullptr;
  double *d_bb = nullptr, *d_dd = nullptr, *d_bd = nullptr;
  DevVec w_x, w_y, w_r, w_p, w_p2, w_Ap, w_b, w_d, w_dinv, w_vpart, w_hist, w_ediag, w_ldiag;
  PcgState* d_state = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  struct Graph {  // cached fixed-iteration PCG graph for one operand set
    std::vector<const void*> key;
    cudaGraphExec_t exec = nullptr;
    int64_t kernels = 0;
  };
  std::vector<Graph> graphs;
  void drop_graphs() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    graphs.clear();
  }
  // pipelined host batches (hxf_pcg_host_batch): copy streams, slot events
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_b[2] = {}, ev_solved[2] = {}, ev_x[2] = {};
  DevVec w_b2, w_x2, w_states, w_hists;
  // partitioned box (hxf_operator_set_partition): the communicator, the
  // subdomains sharing this lattice's low / high face plane per axis, the
  // owner mask over scalar nodes (dots) and plane staging buffers
  hxf::Comm* comm = nullptr;
  int neighbor[3][2] = {{-1, -1}, {-1, -1}, {-1, -1}};
  uint32_t* d_own = nullptr;
  DevVec w_halo;
  // boundary-first apply: elements touching an interface plane, then the
  // rest, while the sum-exchange runs on a high-priority stream
  int* d_elist = nullptr;
  int64_t n_bnd = 0, n_int = 0;
  cudaStream_t s_comm = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;

  int64_t size() const { return int64_t(m) * n_L; }
  Lattice lattice() const {
    Lattice L;
    L.p = p;
    L.S = (p + 1) * (p + 1) * (p + 1);
    L.E = E;
    L.n_L = n_L;
    L.NX = NX;
    L.NY = NY;
    L.nx = nx;
    L.ny = ny;
    L.nz = nz;
    return L;
  }
  ~hxf_op() {
    for (void* ptr : {(void*)d_idx, (void*)d_mask, (void*)d_qd_diff, (void*)d_qd_mass,
                      (void*)d_part, (void*)d_B, (void*)d_G, (void*)d_Bt, (void*)d_Gt,
                      (void*)d_bb, (void*)d_dd, (void*)d_bd, (void*)d_state, (void*)d_own, (void*)d_elist})
      if (ptr) cudaFree(ptr);
    for (DevVec* v : {&w_x, &w_y, &w_r, &w_p, &w_p2, &w_Ap, &w_b, &w_d, &w_dinv, &w_vpart, &w_hist, &w_ediag,
                      &w_ldiag, &w_halo, &w_b2, &w_x2, &w_states, &w_hists})
      v->release();
    for (auto e : ev) cudaEventDestroy(e);
    drop_graphs();
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : {ev_b[k], ev_solved[k], ev_x[k]})
        if (e) cudaEventDestroy(e);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_comm) cudaStreamDestroy(s_comm);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    if (ev_t0) cudaEventDestroy(ev_t0);
    if (ev_t1) cudaEventDestroy(ev_t1);
  }
};

namespace hxf {
// dist.cu: interface sum-exchange and all-reduce for partitioned operators
// (no-ops for a single-domain operator).
void op_halo_sum(hxf_op* op, double* v, cudaStream_t s);
void op_allreduce(hxf_op* op, double* dev, int n, cudaStream_t s);
bool op_partitioned(const hxf_op* op);
bool op_graph_safe(const hxf_op* op);
bool overlap_enabled();  // HXF_OVERLAP=0: exchange after the whole apply
void set_last_error(const char* msg);  // capi.cu: the thread's hxf_last_error()
void op_set_constrained(hxf_op* op, double* v, double value, cudaStream_t s);
}  // namespace hxf

namespace hxf_detail {
// Run f, mapping HxfError / std::exception onto the C status codes (message
// left in the thread's hxf_last_error()).
template <class F>
int guarded(F&& f) {
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

// Structured-box lattice of a restriction (capi.cu): the reference's
// numbering (mesh.cpp:80-104) recognised and verified entry by entry, or the
// implicit box given by dims when idx is NULL.
struct BoxDims {
  int nx = 0, ny = 0, nz = 0;
  int64_t NX = 0, NY = 0, NZ = 0;
};
bool detect_box(int p, int64_t E, int64_t n_L, const int64_t* idx, const int dims[3],
                const char* who, BoxDims* out);
}  // namespace hxf_detail
