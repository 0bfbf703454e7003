// The hxf C-ABI (include/hxf.h): context, operator handle, apply, diagonal,
// restriction / basis / QFunction / geometric-factor entry points and the
// device-resident PCG driver.
//
// Errors are raised internally as HxfError and mapped to the C status codes
// at the boundary, with the reference's own messages where one exists
// (proj/src/operator.cpp:26-46,67-68, pcg.cpp:27-31,54,75-91,
// qfunction.cpp:82-89,120).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cuda.h>

#include "capi_internal.h"

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
int g_sms = 0;

// Lagrange derivative matrix on the q quadrature points (barycentric form,
// evaluated in long double): D[i][j] = l_j'(x_i).  Used for the collocated-
// gradient factorisation of interpolating bases (op_kernel.cuh).
std::vector<double> quad_derivative_matrix(const double* x, int q) {
  std::vector<long double> w(q, 1.0L);
  for (int j = 0; j < q; ++j)
    for (int k = 0; k < q; ++k)
      if (k != j) w[j] *= (long double)x[j] - (long double)x[k];
  std::vector<double> D(size_t(q) * q, 0.0);
  for (int i = 0; i < q; ++i) {
    long double diag = 0.0L;
    for (int j = 0; j < q; ++j) {
      if (j == i) continue;
      const long double v = (w[i] / w[j]) / ((long double)x[i] - (long double)x[j]);
      D[size_t(i) * q + j] = (double)v;
      diag -= v;
    }
    D[size_t(i) * q + i] = (double)diag;
  }
  return D;
}

}  // namespace

namespace hxf {

int num_sms() {
  if (!g_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_sms <= 0) g_sms = 148;
  }
  return g_sms;
}

void count_launch(int n) { g_launches += n; }

int ablate_bits() {
  static const int bits = [] {
    const char* v = std::getenv("HXF_ABLATE");
    return v ? std::atoi(v) : 0;
  }();
  return bits;
}

// HXF_OP_KERNEL (initial value) / hxf_debug_set_op_kernel
std::atomic<int> g_op_choice{[] {
  const char* v = std::getenv("HXF_OP_KERNEL");
  if (!v) return 0;
  const std::string s(v);
  return s == "pencil" ? 1 : (s == "generic" ? 2 : 0);
}()};

int op_kernel_choice() { return g_op_choice.load(std::memory_order_relaxed); }

bool pencil_disabled() {
  // HXF_PENCIL=0: collocated sizes without a tensor-core path on the line kernel (A/B)
  static const bool off = [] {
    const char* v = std::getenv("HXF_PENCIL");
    return v && v[0] == '0';
  }();
  return op_kernel_choice() == 2 || off;
}

bool pdl_apply_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("HXF_PDL_APPLY");
    return v && v[0] == '0';
  }();
  return off;
}

// HXF_STEP_APZ=1: the step kernel zeroes Ap in phase 1 and the DMMA kernel
// stores Ap = p on the constrained rows (measured and dropped: C3 CG iteration
// 156.4 -> 161.2 us, K1 89 -> 93 us; the zeros leave L2 before K1 adds into them)
bool step_ap_zero() {
  static const bool on = [] {
    const char* v = std::getenv("HXF_STEP_APZ");
    return v && v[0] == '1';
  }();
  return on;
}

// HXF_STEP_PDL=1: the operator kernel after a fused step kernel with
// programmatic dependent launch (the step kernel triggers as each CTA ends).
// Measured neutral to slightly worse (C3 CG 156.7 vs 157.4 us): kept off
bool step_pdl() {
  static const bool on = [] {
    const char* v = std::getenv("HXF_STEP_PDL");
    return v && v[0] == '1';
  }();
  return on;
}

bool dmma3_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("HXF_DMMA3");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool dmmaeo_enabled(int P, int ncomp) {
  // measured (BP5 / BP6 ~1e7 DOFs, K1): the even-odd tensor-core kernel wins
  // from p = 12 (one component: p = 12 287 vs 289 us, p = 13 286 vs 366 us,
  // p = 15 198 vs 314 us; p = 11 296 vs 261) and p = 11 (three components:
  // 321 vs 374 us, p = 15 197 vs 410 us); the line / pencil kernels stay ahead below
  static const int mode = [] {
    const char* v = std::getenv("HXF_DMMAEO");
    return v ? std::atoi(v) : 1;
  }();
  if (mode == 0) return false;
  if (mode == 2) return true;  // every P = 9..16 (A/B)
  return ncomp == 1 ? P >= 13 : P >= 12;
}

bool dmma_pad_disabled() {
  static const bool off = [] {
    const char* v = std::getenv("HXF_DMMA_PAD");
    return v && v[0] == '0';
  }();
  return off;
}

bool pdl_enabled() {  // measured neutral in the CG graph at C3: opt-in
  static const bool on = [] {
    const char* v = std::getenv("HXF_PDL");
    return v && v[0] == '1';
  }();
  return on;
}

bool overlap_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("HXF_OVERLAP");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool serpentine() {
  static const bool on = [] {
    const char* v = std::getenv("HXF_SERPENTINE");
    return !(v && v[0] == '0');
  }();
  return on;
}

bool xbatch() {  // HXF_XBATCH=0: x += alpha p every iteration (A/B)
  static const bool on = [] {
    const char* v = std::getenv("HXF_XBATCH");
    return !(v && v[0] == '0');
  }();
  return on;
}

int dmma_stages() {
  static const int ns = [] {
    const char* v = std::getenv("HXF_DMMA_STAGES");
    return (v && v[0] == '2') ? 2 : 1;
  }();
  return ns;
}

int dmma_warps() {
  static const int nw = [] {
    const char* v = std::getenv("HXF_DMMA_NW");
    const int n = v ? std::atoi(v) : 0;
    return (n == 2 || n == 4 || n == 8) ? n : 4;
  }();
  return nw;
}

int max_op_grid() { return num_sms() * 32; }

bool lattice_tma_ok(const OpParams& prm, int m) {
  static const bool off = [] {
    const char* v = std::getenv("HXF_TMA");
    return v && v[0] == '0';
  }();
  if (off || !prm.x || prm.idx) return false;
  if ((reinterpret_cast<uintptr_t>(prm.x) & 15u) != 0) return false;
  if ((prm.NX * 8) % 16 != 0 || (prm.NX * prm.NY * 8) % 16 != 0) return false;
  if (m > 1 && (prm.n_L * 8) % 16 != 0) return false;
  const int64_t lim = int64_t(1) << 31;
  return prm.NX < lim && prm.NY < lim && prm.NZ < lim && m >= 1 && m <= 3;
}

bool encode_lattice_map(const OpParams& prm, int m, void* map_out) {
  using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return Encode(nullptr);
    return reinterpret_cast<Encode>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t dims[4] = {cuuint64_t(prm.NX), cuuint64_t(prm.NY), cuuint64_t(prm.NZ),
                              cuuint64_t(m)};
  const cuuint64_t strides[3] = {cuuint64_t(prm.NX) * 8, cuuint64_t(prm.NX * prm.NY) * 8,
                                 cuuint64_t(prm.n_L) * 8};
  const cuuint32_t box[4] = {12, 8, 8, 1};  // 12 columns from an even start (op_dmma.cuh)
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return encode(static_cast<CUtensorMap*>(map_out), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                const_cast<double*>(prm.x), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
std::atomic<int> g_grid_cap{[] {
  const char* v = std::getenv("HXF_MAX_GRID");
  return v ? std::max(0, std::atoi(v)) : 0;
}()};
}  // namespace
int grid_cap() { return g_grid_cap.load(std::memory_order_relaxed); }

bool centro_symmetric(int P, int Q, bool interp, const double* B, const double* D) {
  auto close = [](double a, double b, double scale) { return std::fabs(a - b) <= 1e-13 * scale; };
  double sb = 0, sd = 0;
  for (int i = 0; i < Q * P; ++i) sb = std::fmax(sb, std::fabs(B[i]));
  for (int i = 0; i < Q * Q; ++i) sd = std::fmax(sd, std::fabs(D[i]));
  for (int o = 0; o < Q; ++o)
    for (int a = 0; a < Q; ++a)
      if (!close(D[(Q - 1 - o) * Q + (Q - 1 - a)], -D[o * Q + a], sd)) return false;
  if (interp)
    for (int o = 0; o < Q; ++o)
      for (int a = 0; a < P; ++a)
        if (!close(B[(Q - 1 - o) * P + (P - 1 - a)], B[o * P + a], sb)) return false;
  return true;
}


cudaError_t launch_op(int P, int Q, int NC, bool interp, int qk, const OpParams& prm,
                      const double* B, const double* D, cudaStream_t s, int* grid_out) {
  switch (P) {
#define HXF_CASE(N) \
  case N:           \
    return launch_op_p##N(Q, NC, interp, qk, prm, B, D, s, grid_out);
    HXF_CASE(2) HXF_CASE(3) HXF_CASE(4) HXF_CASE(5) HXF_CASE(6) HXF_CASE(7) HXF_CASE(8)
    HXF_CASE(9) HXF_CASE(10) HXF_CASE(11) HXF_CASE(12) HXF_CASE(13) HXF_CASE(14) HXF_CASE(15)
    HXF_CASE(16)
#undef HXF_CASE
    default:
      return cudaErrorNotSupported;
  }
}

void set_last_error(const char* msg) { g_err = msg; }

}  // namespace hxf



namespace hxf_detail {

bool detect_box(int p, int64_t E, int64_t n_L, const int64_t* idx, const int dims[3],
                const char* who, BoxDims* out) {
  const int n1 = p + 1;
  const int64_t S = int64_t(n1) * n1 * n1;
  int64_t nx = dims ? dims[0] : 0, ny = dims ? dims[1] : 0, nz = dims ? dims[2] : 0;
  if (!idx) {  // implicit structured box (dims validated here)
    const int64_t NX = nx * p + 1, NY = ny * p + 1, NZ = nz * p + 1;
    if (nx < 1 || ny < 1 || nz < 1 || nx * ny * nz != E || NX * NY * NZ != n_L)
      fail(HXF_EINVAL, std::string(who) + ": dims do not match num_elements / n_L");
    *out = BoxDims{int(nx), int(ny), int(nz), NX, NY, NZ};
    return true;
  }
  if (nx <= 0 || ny <= 0 || nz <= 0) {
    const int64_t NXg = idx[n1];           // node of slot (0,1,0) in element 0
    const int64_t NXNY = idx[n1 * n1];     // node of slot (0,0,1)
    if (NXg <= 1 || (NXg - 1) % p || NXNY % NXg) return false;
    nx = (NXg - 1) / p;
    const int64_t NYg = NXNY / NXg;
    if ((NYg - 1) % p) return false;
    ny = (NYg - 1) / p;
    if (nx * ny == 0 || E % (nx * ny)) return false;
    nz = E / (nx * ny);
  }
  if (nx * ny * nz != E) return false;
  const int64_t NX = nx * p + 1, NY = ny * p + 1, NZ = nz * p + 1;
  if (NX * NY * NZ != n_L) return false;
  for (int64_t e = 0; e < E; ++e) {
    const int64_t ex = e % nx, ey = (e / nx) % ny, ez = e / (nx * ny);
    const int64_t* row = idx + e * S;
    int64_t s = 0;
    for (int kz = 0; kz <= p; ++kz)
      for (int ky = 0; ky <= p; ++ky)
        for (int kx = 0; kx <= p; ++kx, ++s)
          if (row[s] != (ex * p + kx) + NX * ((ey * p + ky) + NY * (ez * p + kz))) return false;
  }
  *out = BoxDims{int(nx), int(ny), int(nz), NX, NY, NZ};
  return true;
}

}  // namespace hxf_detail

namespace {

cudaStream_t pick_stream(hxf_op* op, void* stream) {
  return stream ? static_cast<cudaStream_t>(stream) : op->ctx->stream;
}

// y = op x on the device (y preset here unless zero_y is false; the kernel
// REDs into it).  PCG (st != nullptr): per-CTA partials of p.(A p) go to
// dot_part and the last CTA of the last pass derives alpha into *st.
// Does the operator kernel store y = x on the constrained rows itself when
// asked (prm.cons_store)?  The DMMA kernel (single domain, p = 7 diffusion).
bool k1_stores_cons(const hxf_op* op) {
  return op->P == 8 && !op->interp && op->beta == 0.0 && !op->d_own && op->cons_mode != 0 &&
         op_kernel_choice() == 0;
}

// k1_cons (PCG, fused step): y is all zero and the kernel stores y = x on the
// constrained rows (no preset of them by the step kernel)
void device_apply(hxf_op* op, const double* x, double* y, cudaStream_t s, double* dot_part,
                  int* nparts, const int* stop, bool zero_y = true, PcgState* st = nullptr,
                  bool halo = true, int rev = 0, bool k1_cons = false, bool k1_pdl = false) {
  // single-domain p = 7 collocated diffusion: y zeroed by a write-only memset
  // and the DMMA kernel stores y = x on the constrained rows it gathers
  // (instead of the read-x/write-y init_y pass)
  const bool cons_store = zero_y && k1_stores_cons(op);
  if (cons_store)
    ck(cudaMemsetAsync(y, 0, sizeof(double) * op->n_L * op->m, s), "y memset");
  else if (zero_y)
    ck(launch_init_y(s, op->n_L, op->m, x, y, op->d_mask, op->d_own), "init_y");
  OpParams prm{};
  prm.cons_store = (cons_store || k1_cons) ? 1 : 0;
  // single apply: the kernel's factor copy and setup overlap the memset's tail
  // (it waits in griddepcontrol.wait before touching y); measured 90.6 -> 88.4 us
  prm.pdl = (cons_store && !pdl_apply_disabled()) || (k1_pdl && step_pdl()) ? 1 : 0;
  prm.x = x;
  prm.y = y;
  prm.E = op->E;
  prm.n_L = op->n_L;
  prm.NX = op->NX;
  prm.NY = op->NY;
  prm.NZ = op->NZ;
  prm.nx = op->nx;
  prm.ny = op->ny;
  prm.idx = op->structured ? nullptr : op->d_idx;
  prm.cons_mode = op->cons_mode;
  prm.bnd_faces = op->bnd_faces;
  prm.cons_mask = op->d_mask;
  prm.stop = stop;
  prm.ablate = ablate_bits();
  prm.D = op->d_G;
  prm.rev = rev;
  const int last_pass = op->beta != 0.0 ? 1 : 0;
  int total = 0;
  auto launch = [&](int pass, double coef, PcgState* fin_st) {
    prm.qd = pass == 0 ? op->d_qd_diff : op->d_qd_mass;
    prm.coef = coef;
    prm.dot_partials = dot_part ? dot_part + total : nullptr;
    prm.fin = PcgAlphaFin{fin_st, dot_part, total};
    int grid = 0;
    const cudaError_t err = launch_op(op->P, op->Q, op->m, op->interp, pass == 0 ? 1 : 2, prm,
                                      op->B.data(), op->Dq.data(), s, &grid);
    if (err == cudaErrorNotSupported)
      fail(HXF_EUNSUPPORTED, "operator kernel not instantiated for this (p, q, m)");
    ck(err, "operator kernel launch");
    total += grid;
  };
  // partitioned, one stage (every BP has alpha XOR beta): boundary elements,
  // fork the sum-exchange of the interface planes (only boundary elements
  // touch them) onto the comm stream, interior elements meanwhile, join.
  // Every K1 family takes an element list (DMMA incl. the padded tile,
  // pencil, line); only the general kernel of non-centro-symmetric bases
  // (op_kernel.cuh) does not.
  const bool one_stage = (op->alpha == 0.0) != (op->beta == 0.0);
  const bool elist_ok = op_kernel_choice() != 2 && op->symmetric;
  const bool split = halo && op->comm && op->d_elist && op->n_bnd > 0 && op->n_int > 0 &&
                     one_stage && elist_ok && overlap_enabled();
  if (split) {
    const int pass = op->alpha != 0.0 ? 0 : 1;
    const double coef = pass == 0 ? op->alpha : op->beta;
    prm.elist = op->d_elist;
    prm.E = op->n_bnd;
    launch(pass, coef, nullptr);
    ck(cudaEventRecord(op->ev_fork, s), "fork");
    prm.elist = op->d_elist + op->n_bnd;
    prm.E = op->n_int;
    launch(pass, coef, st);
    ck(cudaStreamWaitEvent(op->s_comm, op->ev_fork, 0), "fork");
    op_halo_sum(op, y, op->s_comm);
    ck(cudaEventRecord(op->ev_join, op->s_comm), "join");
    ck(cudaStreamWaitEvent(s, op->ev_join, 0), "join");
    if (nparts) *nparts = total;
    return;
  }
  for (int pass = 0; pass < 2; ++pass) {
    const double coef = pass == 0 ? op->alpha : op->beta;
    if (coef == 0.0) continue;
    launch(pass, coef, pass == last_pass ? st : nullptr);
  }
  if (nparts) *nparts = total;
  if (halo) op_halo_sum(op, y, s);  // partitioned: assemble interface rows (else no-op)
}

std::vector<int64_t> sorted_unique(const int64_t* v, int64_t n) {
  std::vector<int64_t> out(v, v + n);
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
  return out;
}

// Recognise the reference's structured-box numbering (mesh.cpp:80-104) and
// verify it entry by entry (bit-exact assembly map).  idx == nullptr: the
// implicit box given by dims (checked against E and n_L; `who` names the
// caller in the error message).
bool detect_structured(hxf_op* op, const int64_t* idx, const int dims[3]) {
  BoxDims b;
  if (!detect_box(op->p, op->E, op->n_L, idx, dims, "make_operator", &b)) return false;
  op->nx = b.nx;
  op->ny = b.ny;
  op->nz = b.nz;
  op->NX = b.NX;
  op->NY = b.NY;
  op->NZ = b.NZ;
  return true;
}

void upload_qdata(hxf_op* op, const double* src, int nplanes, hxf_memspace space, double** dst,
                  int64_t* stride) {
  const int64_t Q3 = int64_t(op->q) * op->q * op->q;
  const int64_t w = nplanes * Q3;
  *stride = (w + 1) / 2 * 2;  // 16-byte element blocks for the bulk copy
  *dst = dalloc<double>(size_t(op->E) * *stride + 2);
  ck(cudaMemcpy2DAsync(*dst, size_t(*stride) * 8, src, size_t(w) * 8, size_t(w) * 8,
                       size_t(op->E),
                       space == HXF_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                       op->ctx->stream),
     "qdata upload");
}


// ---------------------------------------------------------------- PCG driver
// One device-resident Jacobi-PCG solve (pcg.cpp:24-115) on op's stream:
// init (x = 0, r = b, p = z, dinv = 1/diag, ||b||, rho) then per iteration
//   K1 (Ap += A p, last CTA: pAp) -> [halo sum Ap, all-reduce pAp]
//   update (alpha; x, r; r.r, r.z) -> [all-reduce] -> direction (beta; p, Ap preset)
struct PcgSolve {
  hxf_op* op;
  const double* db;
  const double* dd;
  double* dx;
  double* dinv;
  int limit;
  bool fixed, timed;
};

double* state_red(hxf_op* op) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(op->d_state) +
                                   offsetof(PcgState, red));
}

void pcg_prepare(hxf_op* op, int limit) {
  if (!op->d_state) op->d_state = dalloc<PcgState>(2);  // [0] live, [1] per-call template
  if (!op->ev_t0) {
    ck(cudaEventCreate(&op->ev_t0), "event");
    ck(cudaEventCreate(&op->ev_t1), "event");
  }
  while (op->ev.size() < size_t(2 * limit)) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    op->ev.push_back(e);
  }
  const size_t n = size_t(op->size());
  // every work buffer a cached solve graph captured by address: growing one
  // (e.g. w_hist for a longer tolerance solve) frees the old allocation, so
  // the graphs holding it are dropped (they would replay into freed memory)
  auto captured = [op] {
    return std::vector<const void*>{op->w_r.p, op->w_p.p, op->w_p2.p, op->w_Ap.p,
                                    op->w_vpart.p, op->w_hist.p, op->w_halo.p};
  };
  const std::vector<const void*> before = captured();
  op->w_r.ensure(n);
  op->w_p.ensure(n);
  if (xbatch()) op->w_p2.ensure(n);
  op->w_Ap.ensure(n);
  op->w_vpart.ensure(size_t(3 * vec_grid()));  // per-CTA partials (<= 3 per CTA)
  op->w_hist.ensure(size_t(limit) + 2);
  if (captured() != before) op->drop_graphs();
}

// the solve's kernels (captured into a graph or run eagerly)
void pcg_enqueue_init(const PcgSolve& ps, cudaStream_t s) {
  hxf_op* op = ps.op;
  ck(pcg_launch_init(s, op->d_state, op->n_L, op->m, ps.db, ps.dd, ps.dinv, ps.dx, op->w_r.p,
                     op->w_p.p, op->w_Ap.p, op->d_mask, op->d_own, op->w_vpart.p),
     "pcg init");
  op_allreduce(op, state_red(op) + 4, 2, s);  // b.b, b.z
  ck(pcg_launch_init_finalize(s, op->d_state, op->w_hist.p), "pcg init");
}

void pcg_enqueue_iteration(const PcgSolve& ps, int it, cudaStream_t s, bool capturing) {
  hxf_op* op = ps.op;
  // batched x updates: p alternates between two buffers (iteration it reads
  // its p from A when odd, B when even) so the previous direction survives
  const bool xb = xbatch();
  double *r = op->w_r.p, *Ap = op->w_Ap.p, *vpart = op->w_vpart.p;
  double* pA = op->w_p.p;
  double* pB = xb ? op->w_p2.p : op->w_p.p;
  double* p = (xb && !(it & 1)) ? pB : pA;
  double* red = state_red(op);
  auto record = [&](cudaEvent_t e) {
    // (External: inside a captured graph the record is a real timing event)
    ck(capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal) : cudaEventRecord(e, s),
       "event");
  };
  // serpentine sweeps: every kernel runs opposite to the one before it, so it
  // starts on the vectors the previous kernel touched last (still in the
  // 126 MB L2); the three-kernel cycle flips each iteration
  const int serp = serpentine() ? 1 : 0, odd = it & 1;
  int nparts = 0;
  if (ps.timed) record(op->ev[2 * (it - 1)]);
  const int xmode = !xb ? 0 : ((it & 1) ? 1 : 2);
  double* pout = !xb ? pA : ((it & 1) ? pB : pA);
  // single domain: update + direction as one cooperative kernel (grid barrier
  // between them, z kept on chip) — no all-reduce has to sit in between; with
  // the DMMA operator kernel storing Ap = p on the constrained rows itself,
  // the step kernel zeroes Ap right after reading it and writes no preset
  const bool fused = !op->comm && !op->d_own &&
                     pcg_step_fusable(op->n_L, ps.dinv, r, ps.dx, p, xmode == 2 ? pA : nullptr, pout, Ap);
  const bool k1c = fused && k1_stores_cons(op) && step_ap_zero();
  // Ap was preset by the init / direction kernel: no memset pass here
  // partitioned: the interface sum-exchange of Ap is part of the apply
  // (overlapped with the interior elements where the kernel allows)
  device_apply(op, p, Ap, s, op->d_part, &nparts, &op->d_state->stop, /*zero_y=*/false,
               op->d_state, /*halo=*/true, serp & (odd ^ 1), k1c, /*k1_pdl=*/fused && it > 1);
  if (ps.timed) record(op->ev[2 * (it - 1) + 1]);  // apply time (single GPU: K1 alone)
  if (fused) {
    ck(pcg_launch_step(s, op->d_state, it, op->w_hist.p, op->n_L, op->m, ps.dinv, r, ps.dx, p,
                       xmode == 2 ? pA : nullptr, pout, Ap, op->d_mask, vpart, serp & odd, xmode,
                       k1c),
       "pcg step");
    return;
  }
  op_allreduce(op, red, 1, s);                     // pAp
  ck(pcg_launch_update(s, op->d_state, it, op->n_L, op->m, ps.dinv, r, Ap, op->d_own, vpart,
                       serp & odd),
     "pcg update");
  op_allreduce(op, red + 1, 2, s);  // r.r, r.z
  ck(pcg_launch_direction(s, op->d_state, it, op->w_hist.p, op->n_L, op->m, ps.dinv, r, ps.dx, p,
                          xmode == 2 ? pA : nullptr, pout, Ap, op->d_mask, op->d_own, vpart,
                          serp & (odd ^ 1), xmode),
     "pcg direction");
}

// fixed-iteration solve as one CUDA graph (launch-gap free), captured once per
// operand set and replayed; a small per-operator cache serves alternating
// operand sets (pipelined batches)
void pcg_launch_fixed_graph(const PcgSolve& ps, cudaStream_t s) {
  hxf_op* op = ps.op;
  const std::vector<const void*> key = {ps.db, ps.dd, ps.dx, ps.dinv,
                                        (const void*)(intptr_t)ps.limit,
                                        (const void*)(intptr_t)ps.timed, (const void*)s};
  hxf_op::Graph* g = nullptr;
  for (auto& cand : op->graphs)
    if (cand.key == key) g = &cand;
  if (!g) {
    if (op->graphs.size() >= 4) {
      cudaGraphExecDestroy(op->graphs.front().exec);
      op->graphs.erase(op->graphs.begin());
    }
    hxf_op::Graph ng;
    ng.key = key;
    const int64_t before = hxf_launch_count();
    cudaGraph_t graph;
    ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed), "capture");
    pcg_enqueue_init(ps, s);
    for (int it = 1; it <= ps.limit; ++it) pcg_enqueue_iteration(ps, it, s, true);
    ck(cudaStreamEndCapture(s, &graph), "capture");
    const cudaError_t ierr = cudaGraphInstantiate(&ng.exec, graph, 0);
    cudaGraphDestroy(graph);
    ck(ierr, "graph instantiate");
    ng.kernels = hxf_launch_count() - before;
    count_launch(-int(ng.kernels));  // counted on replay below
    op->graphs.push_back(ng);
    g = &op->graphs.back();
  }
  ck(cudaGraphLaunch(g->exec, s), "graph launch");
  count_launch(int(g->kernels));
}

// Enqueue a whole solve; tolerance mode polls the stop flag every few
// iterations (host sync), fixed mode never syncs.  Returns iterations launched.
int pcg_enqueue_solve(const PcgSolve& ps, cudaStream_t s) {
  hxf_op* op = ps.op;
  // per-call template state (uploaded by the caller) -> live state
  ck(cudaMemcpyAsync(op->d_state, op->d_state + 1, sizeof(PcgState), cudaMemcpyDeviceToDevice, s),
     "state");
  if (ps.fixed && op_graph_safe(op)) {
    pcg_launch_fixed_graph(ps, s);
    return ps.limit;
  }
  pcg_enqueue_init(ps, s);
  if (ps.fixed) {  // host-synchronous communicator: no graph capture
    for (int it = 1; it <= ps.limit; ++it) pcg_enqueue_iteration(ps, it, s, false);
    return ps.limit;
  }
  int launched = 0;
  PcgState hs{};
  ck(cudaMemcpyAsync(&hs, op->d_state, sizeof hs, cudaMemcpyDeviceToHost, s), "state");
  ck(cudaStreamSynchronize(s), "pcg init");
  while (!hs.stop && launched < ps.limit) {
    const int chunk = std::min(ps.limit - launched, launched < 4 ? 1 : 8);
    for (int i = 0; i < chunk; ++i) pcg_enqueue_iteration(ps, ++launched, s, false);
    ck(cudaMemcpyAsync(&hs, op->d_state, sizeof hs, cudaMemcpyDeviceToHost, s), "state");
    ck(cudaStreamSynchronize(s), "pcg");
  }
  return launched;
}

void pcg_upload_template(hxf_op* op, const hxf_pcg_options* opts, int limit, bool fixed,
                         cudaStream_t s) {
  PcgState st{};
  st.tol = opts->tol_rel;
  st.limit = limit;
  st.fixed = fixed ? 1 : 0;
  h2d(op->d_state + 1, &st, sizeof st, s);
}

void pcg_fill_report(hxf_op* op, const PcgState& hs, const double* hist_dev, int launched,
                     bool timed, hxf_solve_report* report) {
  if (hs.error) {
    static const char* msgs[] = {"", "pcg: right-hand side is not finite",
                                 "pcg: NaN in operator apply",
                                 "pcg: indefinite direction (p^T A p <= 0), operator is not SPD",
                                 "pcg: residual is not finite"};
    fail(HXF_ENUMERIC, msgs[hs.error]);
  }
  const int iters = hs.it;
  report->iterations = iters;
  report->converged = (hs.converged || hs.res <= hs.target) ? 1 : 0;
  if (report->residual_history && report->history_capacity > 0) {
    const int nh = std::min(report->history_capacity, iters + 1);
    ck(cudaMemcpy(report->residual_history, hist_dev, size_t(nh) * 8, cudaMemcpyDeviceToHost),
       "history");
  }
  double apply_ms = 0;
  for (int i = 0; timed && i < std::min(iters, launched); ++i) {
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, op->ev[2 * i], op->ev[2 * i + 1]), "elapsed");
    apply_ms += ms;
  }
  report->apply_time_seconds = apply_ms * 1e-3;
}

}  // namespace

extern "C" {


const char* hxf_last_error(void) { return g_err.c_str(); }
int hxf_abi_version(void) { return HXF_ABI_VERSION; }
int64_t hxf_launch_count(void) { return g_launches.load(); }

int hxf_debug_set_grid_cap(int cap) {
  const int old = g_grid_cap.load();
  g_grid_cap.store(cap > 0 ? cap : 0);
  return old;
}

int hxf_debug_set_op_kernel(int choice) {
  return g_op_choice.exchange(choice == 1 || choice == 2 ? choice : 0);
}

int hxf_debug_step_timestamps(int on, unsigned long long* out) {
  return guarded([&] { pcg_step_timestamps(on, out); });
}

int hxf_context_create(int device, void* nccl_comm, hxf_ctx** out) {
  return guarded([&] {
    if (!out) fail(HXF_EINVAL, "hxf_context_create: out is NULL");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      fail(HXF_ECUDA, "hxf: no CUDA device (there is no CPU fallback)");
    if (device < 0 || device >= n) fail(HXF_EINVAL, "hxf_context_create: bad device ordinal");
    ck(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp prop{};
    ck(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
    if (prop.major != 10)
      fail(HXF_ECUDA, "hxf kernels are compiled for sm_100a (B200); device is sm_" +
                          std::to_string(prop.major) + std::to_string(prop.minor));
    auto* c = new hxf_ctx();
    c->device = device;
    c->nccl = nccl_comm;
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    g_sms = prop.multiProcessorCount;
    *out = c;
  });
}

int hxf_context_destroy(hxf_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->stream);
    for (DevVec* v : {&ctx->scratch_a, &ctx->scratch_b, &ctx->scratch_c, &ctx->scratch_d})
      v->release();
    cudaStreamDestroy(ctx->stream);
    delete ctx;
  });
}

void* hxf_context_stream(hxf_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int hxf_malloc(hxf_ctx* ctx, uint64_t bytes, void** out) {
  return guarded([&] {
    if (!ctx || !out) fail(HXF_EINVAL, "hxf_malloc: NULL argument");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    *out = nullptr;
    ck(cudaMalloc(out, bytes ? bytes : 1), "cudaMalloc");
  });
}

int hxf_free(hxf_ctx* ctx, void* ptr) {
  return guarded([&] {
    if (!ctx) fail(HXF_EINVAL, "hxf_free: NULL context");
    if (ptr) {
      ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
      ck(cudaFree(ptr), "cudaFree");
    }
  });
}

int hxf_memcpy(hxf_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind) {
  return guarded([&] {
    if (!ctx || (!dst && bytes) || (!src && bytes)) fail(HXF_EINVAL, "hxf_memcpy: NULL argument");
    const cudaMemcpyKind k = kind == 0   ? cudaMemcpyHostToDevice
                             : kind == 1 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    ck(cudaMemcpyAsync(dst, src, bytes, k, ctx->stream), "cudaMemcpyAsync");
    ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  });
}

int hxf_synchronize(hxf_ctx* ctx) {
  return guarded([&] {
    if (!ctx) fail(HXF_EINVAL, "hxf_synchronize: NULL context");
    ck(cudaStreamSynchronize(ctx->stream), "cudaStreamSynchronize");
  });
}

int hxf_operator_create(hxf_ctx* ctx, const hxf_operator_desc* d, hxf_op** out) {
  return guarded([&] {
    if (!ctx || !d || !out) fail(HXF_EINVAL, "hxf_operator_create: NULL argument");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    if (d->alpha < 0 || d->beta < 0 || (d->alpha == 0 && d->beta == 0))
      fail(HXF_EINVAL, "make_operator: alpha, beta must be >= 0 and not both zero");
    if (d->p < 1 || d->q < 1 || d->m < 1 || d->num_elements < 1 || d->n_L < 1)
      fail(HXF_EINVAL, "make_operator: restriction/basis size mismatch");
    if (!d->interp1d || !d->grad1d)
      fail(HXF_EINVAL, "make_operator: basis tables are required");
    if (!d->indices && (d->dims[0] < 1 || d->dims[1] < 1 || d->dims[2] < 1))
      fail(HXF_EINVAL, "make_operator: indices (or structured-box dims) are required");
    if (d->beta > 0 && !d->mass_qdata) fail(HXF_EINVAL, "make_operator: mass qdata required");
    if (d->alpha > 0 && !d->diff_qdata)
      fail(HXF_EINVAL, "make_operator: diffusion qdata required");
    auto op = std::make_unique<hxf_op>();
    op->ctx = ctx;
    op->p = d->p;
    op->q = d->q;
    op->m = d->m;
    op->P = d->p + 1;
    op->Q = d->q;
    op->E = d->num_elements;
    op->n_L = d->n_L;
    op->alpha = d->alpha;
    op->beta = d->beta;
    const int n1 = d->p + 1, q = d->q;
    const int64_t S = int64_t(n1) * n1 * n1;
    if (op->P > 16) fail(HXF_EUNSUPPORTED, "hxf: p > 15 has no compiled kernel");
    // element indices run through 32-bit fast division in the operator kernels
    if (op->E >= (int64_t(1) << 31)) fail(HXF_EUNSUPPORTED, "hxf: 2^31 or more elements");
    if (d->indices)
      for (int64_t i = 0; i < op->E * S; ++i)
        if (d->indices[i] < 0 || d->indices[i] >= d->n_L)
          fail(HXF_EINVAL, "make_operator: restriction index out of range");
    std::vector<int64_t> cons;
    if (d->n_constrained > 0) {
      if (!d->constrained) fail(HXF_EINVAL, "make_operator: constrained list is NULL");
      cons = sorted_unique(d->constrained, d->n_constrained);
      if (cons.front() < 0 || cons.back() >= d->n_L)
        fail(HXF_EINVAL, "make_operator: constrained index out of range");
    }
    // basis: collocated (interp1d == I exactly) or interpolating with q = p+2
    bool ident = q == n1;
    for (int i = 0; ident && i < q; ++i)
      for (int j = 0; j < n1; ++j)
        if (d->interp1d[i * n1 + j] != (i == j ? 1.0 : 0.0)) {
          ident = false;
          break;
        }
    op->B.assign(d->interp1d, d->interp1d + size_t(q) * n1);
    if (ident) {
      op->interp = false;
      op->Dq.assign(d->grad1d, d->grad1d + size_t(q) * n1);
    } else if (q == n1 + 1) {
      if (!d->qpoints) fail(HXF_EINVAL, "make_operator: quadrature points required (q != p+1)");
      op->interp = true;
      op->Dq = quad_derivative_matrix(d->qpoints, q);
    } else {
      fail(HXF_EUNSUPPORTED, "hxf: basis needs q = p+1 collocated GLL or q = p+2");
    }
    op->symmetric = centro_symmetric(op->P, op->Q, op->interp, op->B.data(), op->Dq.data());
    // restriction: structured lattice or int32 table
    op->structured = detect_structured(op.get(), d->indices, d->dims);
    if (!op->structured) {
      if (d->n_L >= (int64_t(1) << 31)) fail(HXF_EUNSUPPORTED, "hxf: n_L >= 2^31 with a table");
      std::vector<int> idx32(size_t(op->E * S));
      for (size_t i = 0; i < idx32.size(); ++i) idx32[i] = int(d->indices[i]);
      op->d_idx = dalloc<int>(idx32.size());
      ck(cudaMemcpy(op->d_idx, idx32.data(), idx32.size() * sizeof(int), cudaMemcpyHostToDevice),
         "index upload");
    }
    // constraints: box boundary (computed in the kernel) or bitmask
    op->ncons = int64_t(cons.size());
    if (!cons.empty()) {
      std::vector<uint32_t> mask(size_t((d->n_L + 31) / 32), 0u);
      for (int64_t c : cons) mask[size_t(c >> 5)] |= 1u << (c & 31);
      op->d_mask = dalloc<uint32_t>(mask.size());
      ck(cudaMemcpy(op->d_mask, mask.data(), mask.size() * 4, cudaMemcpyHostToDevice),
         "mask upload");
      op->cons_mode = 2;
      if (op->structured) {
        // box-face form: the list is exactly the union of some faces of the
        // lattice (all six: the single-domain BP3-6 case; a subset: a
        // subdomain of a partitioned box, constrained only on global faces)
        auto bit = [&](int64_t n) { return (mask[size_t(n >> 5)] >> (n & 31)) & 1u; };
        const int64_t NX = op->NX, NY = op->NY, NZ = op->NZ;
        auto face_full = [&](int f) {
          const int axis = f / 2;
          const int64_t fixed = (f & 1) ? (axis == 0 ? NX : axis == 1 ? NY : NZ) - 1 : 0;
          const int64_t na = axis == 0 ? NY : NX, nb = axis == 2 ? NY : NZ;
          for (int64_t b = 0; b < nb; ++b)
            for (int64_t a = 0; a < na; ++a) {
              const int64_t ix = axis == 0 ? fixed : a, iy = axis == 1 ? fixed : (axis == 0 ? a : b),
                            iz = axis == 2 ? fixed : b;
              if (!bit(ix + NX * (iy + NY * iz))) return false;
            }
          return true;
        };
        int faces = 0;
        for (int f = 0; f < 6; ++f)
          if (face_full(f)) faces |= 1 << f;
        OpParams probe{};
        probe.NX = NX;
        probe.NY = NY;
        probe.NZ = NZ;
        probe.bnd_faces = faces;
        bool exact = faces != 0;
        for (size_t i = 0; exact && i < cons.size(); ++i) {
          const int64_t c = cons[i];
          exact = on_bnd_face(probe, c % NX, (c / NX) % NY, c / (NX * NY));
        }
        if (exact) {
          op->cons_mode = 1;
          op->bnd_faces = faces;
        }
      }
    }
    if (op->alpha > 0) upload_qdata(op.get(), d->diff_qdata, 6, d->qdata_space, &op->d_qd_diff,
                                    &op->diff_stride);
    if (op->beta > 0) upload_qdata(op.get(), d->mass_qdata, 1, d->qdata_space, &op->d_qd_mass,
                                   &op->mass_stride);
    op->d_part = dalloc<double>(size_t(2 * max_op_grid()));
    // 1-D tables for the setup / API-surface kernels
    std::vector<double> Bt(size_t(q) * n1), Gt(size_t(q) * n1), bb(Bt.size()), dd(Bt.size()),
        bd(Bt.size());
    for (int iq = 0; iq < q; ++iq)
      for (int j = 0; j < n1; ++j) {
        Bt[size_t(j) * q + iq] = d->interp1d[iq * n1 + j];
        Gt[size_t(j) * q + iq] = d->grad1d[iq * n1 + j];
      }
    for (size_t i = 0; i < Bt.size(); ++i) {
      bb[i] = Bt[i] * Bt[i];
      dd[i] = Gt[i] * Gt[i];
      bd[i] = Bt[i] * Gt[i];
    }
    auto up = [&](const double* src, size_t n) {
      double* p = dalloc<double>(n);
      ck(cudaMemcpy(p, src, n * 8, cudaMemcpyHostToDevice), "table upload");
      return p;
    };
    op->d_B = up(d->interp1d, Bt.size());
    op->d_G = up(d->grad1d, Bt.size());
    op->d_Bt = up(Bt.data(), Bt.size());
    op->d_Gt = up(Gt.data(), Bt.size());
    op->d_bb = up(bb.data(), Bt.size());
    op->d_dd = up(dd.data(), Bt.size());
    op->d_bd = up(bd.data(), Bt.size());
    ck(cudaStreamSynchronize(ctx->stream), "operator create");
    *out = op.release();
  });
}

int hxf_operator_destroy(hxf_op* op) {
  return guarded([&] {
    if (!op) return;
    cudaStreamSynchronize(op->ctx->stream);
    delete op;
  });
}

int64_t hxf_operator_size(const hxf_op* op) { return op ? op->size() : 0; }
int hxf_operator_is_structured(const hxf_op* op) { return op && op->structured ? 1 : 0; }

int hxf_operator_apply(hxf_op* op, const double* x, double* y, hxf_memspace space, void* stream) {
  return guarded([&] {
    if (!op || !x || !y) fail(HXF_EINVAL, "operator_apply: shape mismatch");
    cudaStream_t s = pick_stream(op, stream);
    const size_t n = size_t(op->size());
    if (space == HXF_DEVICE) {
      device_apply(op, x, y, s, nullptr, nullptr, nullptr);
      ck(cudaGetLastError(), "operator_apply");
      return;
    }
    double* dx = op->w_x.ensure(n);
    double* dy = op->w_y.ensure(n);
    h2d(dx, x, n * 8, s);
    device_apply(op, dx, dy, s, nullptr, nullptr, nullptr);
    d2h(y, dy, n * 8, s);
    ck(cudaStreamSynchronize(s), "operator_apply");
  });
}

int hxf_operator_diagonal(hxf_op* op, double* d, hxf_memspace space) {
  return guarded([&] {
    if (!op || !d) fail(HXF_EINVAL, "operator_diagonal: NULL argument");
    cudaStream_t s = op->ctx->stream;
    const Lattice L = op->lattice();
    double* ediag = op->w_ediag.ensure(size_t(op->E) * L.S);
    double* ldiag = op->w_ldiag.ensure(size_t(op->n_L));
    double* dd = space == HXF_DEVICE ? d : op->w_y.ensure(size_t(op->size()));
    ck(launch_diagonal(s, L, op->structured ? nullptr : op->d_idx, op->structured, op->q, op->d_bb,
                       op->d_dd, op->d_bd, op->d_qd_mass, op->mass_stride, op->d_qd_diff,
                       op->diff_stride, op->alpha, op->beta, op->m, op->d_mask, ediag, ldiag, dd),
       "operator_diagonal");
    if (op_partitioned(op)) {  // one copy of each constrained 1, then assemble
      op_set_constrained(op, dd, 1.0, s);
      op_halo_sum(op, dd, s);
    }
    if (space == HXF_HOST) d2h(d, dd, size_t(op->size()) * 8, s);
    ck(cudaStreamSynchronize(s), "operator_diagonal");
  });
}

int hxf_restriction_apply(hxf_op* op, int transpose, const double* in, double* out,
                          hxf_memspace space) {
  return guarded([&] {
    if (!op || !in || !out) fail(HXF_EINVAL, "apply_g: NULL argument");
    cudaStream_t s = op->ctx->stream;
    const Lattice L = op->lattice();
    const size_t nl = size_t(op->m) * op->n_L, ne = size_t(op->m) * op->E * L.S;
    const size_t nin = transpose ? ne : nl, nout = transpose ? nl : ne;
    const double* din = in;
    double* dout = out;
    if (space == HXF_HOST) {
      double* a = op->ctx->scratch_a.ensure(nin);
      h2d(a, in, nin * 8, s);
      din = a;
      dout = op->ctx->scratch_b.ensure(nout);
    }
    ck(launch_restriction(s, L, op->structured ? nullptr : op->d_idx, op->structured, op->m,
                          transpose != 0, din, dout),
       "restriction");
    if (space == HXF_HOST) d2h(out, dout, nout * 8, s);
    ck(cudaStreamSynchronize(s), "restriction");
  });
}

int hxf_restriction_multiplicity(hxf_op* op, double* out, hxf_memspace space) {
  return guarded([&] {
    if (!op || !out) fail(HXF_EINVAL, "multiplicity: NULL argument");
    cudaStream_t s = op->ctx->stream;
    double* dout = space == HXF_DEVICE ? out : op->ctx->scratch_b.ensure(size_t(op->n_L));
    ck(launch_multiplicity(s, op->lattice(), op->structured ? nullptr : op->d_idx, dout),
       "multiplicity");
    if (space == HXF_HOST) d2h(out, dout, size_t(op->n_L) * 8, s);
    ck(cudaStreamSynchronize(s), "multiplicity");
  });
}

int hxf_basis_apply(hxf_ctx* ctx, int p, int q, const double* interp1d, const double* grad1d,
                    hxf_eval_mode mode, hxf_eval_dir dir, int64_t ne, const double* in,
                    double* out, hxf_memspace space) {
  return guarded([&] {
    if (!ctx || !interp1d || !grad1d || !in || !out)
      fail(HXF_EINVAL, "apply_basis_batch: NULL argument");
    if (p < 1 || q < 1 || p > 16 || q > 17) fail(HXF_EINVAL, "apply_basis_batch: bad p/q");
    cudaStream_t s = ctx->stream;
    const int n1 = p + 1;
    const size_t msz = size_t(q) * n1;
    std::vector<double> tabs(4 * msz);
    std::memcpy(tabs.data(), interp1d, msz * 8);
    std::memcpy(tabs.data() + msz, grad1d, msz * 8);
    for (int iq = 0; iq < q; ++iq)
      for (int j = 0; j < n1; ++j) {
        tabs[2 * msz + size_t(j) * q + iq] = interp1d[iq * n1 + j];
        tabs[3 * msz + size_t(j) * q + iq] = grad1d[iq * n1 + j];
      }
    double* dt = ctx->scratch_c.ensure(tabs.size());
    h2d(dt, tabs.data(), tabs.size() * 8, s);
    const int64_t nd3 = int64_t(n1) * n1 * n1, nq3 = int64_t(q) * q * q;
    const int64_t in_e = (mode == HXF_GRAD && dir == HXF_TRANSPOSE) ? 3 * nq3
                         : (dir == HXF_FORWARD ? nd3 : nq3);
    const int64_t out_e = (mode == HXF_GRAD && dir == HXF_FORWARD) ? 3 * nq3
                          : (dir == HXF_FORWARD ? nq3 : nd3);
    const double* din = in;
    double* dout = out;
    if (space == HXF_HOST) {
      double* a = ctx->scratch_a.ensure(size_t(ne * in_e));
      h2d(a, in, size_t(ne * in_e) * 8, s);
      din = a;
      dout = ctx->scratch_b.ensure(size_t(ne * out_e));
    }
    ck(launch_basis_apply(s, p, q, dt, dt + msz, dt + 2 * msz, dt + 3 * msz, int(mode), int(dir),
                          ne, din, dout),
       "apply_basis_batch");
    if (space == HXF_HOST) d2h(out, dout, size_t(ne * out_e) * 8, s);
    ck(cudaStreamSynchronize(s), "apply_basis_batch");
  });
}

int hxf_qfunction_apply(hxf_ctx* ctx, hxf_qdata_kind kind, const double* qdata,
                        int64_t num_elements, int nq, int64_t e0, int64_t ne, const double* in,
                        double* out, hxf_memspace space) {
  return guarded([&] {
    if (!ctx || !qdata || !in || !out) fail(HXF_EINVAL, "apply_qf: NULL argument");
    if (e0 < 0 || ne < 0 || e0 + ne > num_elements)
      fail(HXF_EINVAL, kind == HXF_QDATA_MASS ? "apply_qf_mass: shape mismatch"
                                              : "apply_qf_diffusion: shape mismatch");
    cudaStream_t s = ctx->stream;
    const int K = kind == HXF_QDATA_MASS ? 1 : 3;
    const int Kq = kind == HXF_QDATA_MASS ? 1 : 6;
    const size_t nio = size_t(K) * ne * nq;
    const double* dq = qdata;
    const double* din = in;
    double* dout = out;
    int64_t ebase = e0;
    if (space == HXF_HOST) {
      double* q = ctx->scratch_c.ensure(size_t(Kq) * ne * nq);
      h2d(q, qdata + size_t(e0) * Kq * nq, size_t(Kq) * ne * nq * 8, s);
      dq = q;
      ebase = 0;
      double* a = ctx->scratch_a.ensure(nio);
      h2d(a, in, nio * 8, s);
      din = a;
      dout = ctx->scratch_b.ensure(nio);
    }
    ck(launch_qfunction(s, kind == HXF_QDATA_MASS ? 0 : 1, dq, nq, ebase, ne, din, dout),
       "apply_qf");
    if (space == HXF_HOST) d2h(out, dout, nio * 8, s);
    ck(cudaStreamSynchronize(s), "apply_qf");
  });
}

int hxf_qdata_compute(hxf_ctx* ctx, int p, int q, const double* interp1d, const double* grad1d,
                      const double* qweights, int64_t num_elements, int64_t n_L,
                      const double* coords, const int64_t* indices, const int dims[3],
                      hxf_qdata_kind kind, double* out, hxf_memspace space) {
  return guarded([&] {
    if (!ctx || !interp1d || !grad1d || !qweights || !coords || !out)
      fail(HXF_EINVAL, "compute_qdata: NULL argument");
    if (p < 1 || q < 1 || p > 16 || q > 17) fail(HXF_EINVAL, "compute_qdata: bad p/q");
    cudaStream_t s = ctx->stream;
    const int n1 = p + 1;
    const int64_t S = int64_t(n1) * n1 * n1, nq = int64_t(q) * q * q;
    Lattice L{};
    L.p = p;
    L.S = int(S);
    L.E = num_elements;
    L.n_L = n_L;
    int* d_idx = nullptr;
    if (indices) {
      std::vector<int> idx32(size_t(num_elements * S));
      for (size_t i = 0; i < idx32.size(); ++i) idx32[i] = int(indices[i]);
      d_idx = dalloc<int>(idx32.size());
      h2d(d_idx, idx32.data(), idx32.size() * 4, s);
    } else {
      if (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1 ||
          int64_t(dims[0]) * dims[1] * dims[2] != num_elements)
        fail(HXF_EINVAL, "compute_qdata: dims required without an index table");
      L.nx = dims[0];
      L.ny = dims[1];
      L.nz = dims[2];
      L.NX = int64_t(dims[0]) * p + 1;
      L.NY = int64_t(dims[1]) * p + 1;
    }
    const size_t msz = size_t(q) * n1;
    std::vector<double> tabs(2 * msz + size_t(q));
    std::memcpy(tabs.data(), interp1d, msz * 8);
    std::memcpy(tabs.data() + msz, grad1d, msz * 8);
    std::memcpy(tabs.data() + 2 * msz, qweights, size_t(q) * 8);
    double* dt = ctx->scratch_c.ensure(tabs.size());
    h2d(dt, tabs.data(), tabs.size() * 8, s);
    const double* dcoords = coords;
    if (space == HXF_HOST) {
      double* c = ctx->scratch_a.ensure(size_t(3 * n_L));
      h2d(c, coords, size_t(3 * n_L) * 8, s);
      dcoords = c;
    }
    const int K = kind == HXF_QDATA_MASS ? 1 : 6;
    double* dout = space == HXF_DEVICE ? out : ctx->scratch_b.ensure(size_t(num_elements * K * nq));
    const int64_t batch = std::max<int64_t>(1, (int64_t(256) << 20) / (9 * nq * 8));
    double* scratch = ctx->scratch_d.ensure(size_t(9 * std::min(batch, num_elements) * nq));
    unsigned long long* fkey = dalloc<unsigned long long>(1);
    double* fdet = dalloc<double>(1);
    const unsigned long long init = ~0ull;
    h2d(fkey, &init, 8, s);
    ck(launch_qdata(s, L, d_idx, q, dt, dt + msz, dt + 2 * msz, dcoords, kind == HXF_QDATA_MASS ? 0 : 1,
                    dout, scratch, std::min(batch, num_elements), fkey, fdet),
       "compute_qdata");
    unsigned long long key = 0;
    double det = 0;
    d2h(&key, fkey, 8, s);
    d2h(&det, fdet, 8, s);
    if (space == HXF_HOST) d2h(out, dout, size_t(num_elements * K * nq) * 8, s);
    ck(cudaStreamSynchronize(s), "compute_qdata");
    cudaFree(fkey);
    cudaFree(fdet);
    if (d_idx) cudaFree(d_idx);
    if (key != ~0ull) {
      char buf[256];
      std::snprintf(buf, sizeof buf,
                    "compute_qdata: non-positive Jacobian determinant (%f) in element %lld at "
                    "quadrature point %lld",
                    det, (long long)(key / nq), (long long)(key % nq));
      fail(HXF_ENUMERIC, buf);
    }
  });
}

int hxf_pcg(hxf_op* op, const double* b, const double* diag, const hxf_pcg_options* opts,
            double* x, hxf_memspace space, hxf_solve_report* report) {
  return guarded([&] {
    if (!op || !b || !x || !opts || !report) fail(HXF_EINVAL, "pcg: vector length mismatch");
    cudaStream_t s = op->ctx->stream;
    const size_t n = size_t(op->size());
    const bool fixed = opts->fixed_iterations >= 0;
    const int limit = fixed ? opts->fixed_iterations : opts->max_iter;
    if (limit < 0) fail(HXF_EINVAL, "pcg: negative iteration limit");
    pcg_prepare(op, limit);
    PcgSolve ps{op, b, diag, x, nullptr, limit, fixed, opts->time_apply != 0};
    if (space == HXF_HOST) {
      double* tb = op->w_b.ensure(n);
      h2d(tb, b, n * 8, s);
      ps.db = tb;
      if (diag) {
        double* td = op->w_d.ensure(n);
        h2d(td, diag, n * 8, s);
        ps.dd = td;
      }
      ps.dx = op->w_x.ensure(n);
    }
    ps.dinv = ps.dd ? op->w_dinv.ensure(n) : nullptr;  // 1/diag, filled by the init kernel
    ck(cudaEventRecord(op->ev_t0, s), "event");
    pcg_upload_template(op, opts, limit, fixed, s);
    const int launched = pcg_enqueue_solve(ps, s);
    ck(cudaEventRecord(op->ev_t1, s), "event");
    PcgState hs{};
    ck(cudaMemcpyAsync(&hs, op->d_state, sizeof hs, cudaMemcpyDeviceToHost, s), "state");
    if (space == HXF_HOST) d2h(x, ps.dx, n * 8, s);
    ck(cudaStreamSynchronize(s), "pcg");
    pcg_fill_report(op, hs, op->w_hist.p, launched, ps.timed, report);
    float tot = 0;
    ck(cudaEventElapsedTime(&tot, op->ev_t0, op->ev_t1), "elapsed");
    report->total_time_seconds = tot * 1e-3;
  });
}

int hxf_pcg_host_batch(hxf_op* op, int nrhs, const double* const* b, const double* diag,
                       const hxf_pcg_options* opts, double* const* x, hxf_solve_report* reports) {
  return guarded([&] {
    if (!op || nrhs < 0 || (nrhs > 0 && (!b || !x || !reports)) || !opts)
      fail(HXF_EINVAL, "pcg_host_batch: NULL argument");
    if (nrhs == 0) return;
    cudaStream_t s = op->ctx->stream;
    const size_t n = size_t(op->size());
    const bool fixed = opts->fixed_iterations >= 0;
    const int limit = fixed ? opts->fixed_iterations : opts->max_iter;
    if (limit < 0) fail(HXF_EINVAL, "pcg: negative iteration limit");
    pcg_prepare(op, limit);
    if (!op->s_h2d) {
      ck(cudaStreamCreateWithFlags(&op->s_h2d, cudaStreamNonBlocking), "stream");
      ck(cudaStreamCreateWithFlags(&op->s_d2h, cudaStreamNonBlocking), "stream");
      for (int k = 0; k < 2; ++k)
        for (cudaEvent_t* e : {&op->ev_b[k], &op->ev_solved[k], &op->ev_x[k]})
          ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    }
    double* dinv = diag ? op->w_dinv.ensure(n) : nullptr;
    double* db[2] = {op->w_b.ensure(n), op->w_b2.ensure(n)};
    double* dx[2] = {op->w_x.ensure(n), op->w_x2.ensure(n)};
    // per-solve state + history snapshots, read back once at the end
    const size_t hstride = size_t(limit) + 2;
    double* states = op->w_states.ensure(size_t(nrhs) * (sizeof(PcgState) / 8 + 1) + 1);
    double* hists = op->w_hists.ensure(size_t(nrhs) * hstride);
    const size_t sst = sizeof(PcgState) / 8 + 1;
    ck(cudaEventRecord(op->ev_t0, s), "event");
    pcg_upload_template(op, opts, limit, fixed, s);
    std::vector<int> launched(static_cast<size_t>(nrhs), 0);
    // three engines: H2D of b(k+1) and D2H of x(k-1) run under solve k
    for (int k = 0; k < nrhs; ++k) {
      const int sl = k & 1;
      if (k >= 2) ck(cudaStreamWaitEvent(op->s_h2d, op->ev_solved[sl], 0), "wait");
      ck(cudaMemcpyAsync(db[sl], b[k], n * 8, cudaMemcpyHostToDevice, op->s_h2d), "H2D b");
      ck(cudaEventRecord(op->ev_b[sl], op->s_h2d), "event");
      ck(cudaStreamWaitEvent(s, op->ev_b[sl], 0), "wait");
      if (k >= 2) ck(cudaStreamWaitEvent(s, op->ev_x[sl], 0), "wait");
      PcgSolve ps{op, db[sl], diag, dx[sl], dinv, limit, fixed, false};
      launched[size_t(k)] = pcg_enqueue_solve(ps, s);
      ck(cudaMemcpyAsync(states + size_t(k) * sst, op->d_state, sizeof(PcgState),
                         cudaMemcpyDeviceToDevice, s),
         "state");
      ck(cudaMemcpyAsync(hists + size_t(k) * hstride, op->w_hist.p, hstride * 8,
                         cudaMemcpyDeviceToDevice, s),
         "history");
      ck(cudaEventRecord(op->ev_solved[sl], s), "event");
      ck(cudaStreamWaitEvent(op->s_d2h, op->ev_solved[sl], 0), "wait");
      ck(cudaMemcpyAsync(x[k], dx[sl], n * 8, cudaMemcpyDeviceToHost, op->s_d2h), "D2H x");
      ck(cudaEventRecord(op->ev_x[sl], op->s_d2h), "event");
    }
    ck(cudaStreamWaitEvent(s, op->ev_x[(nrhs - 1) & 1], 0), "wait");
    ck(cudaEventRecord(op->ev_t1, s), "event");
    ck(cudaStreamSynchronize(s), "pcg batch");
    ck(cudaStreamSynchronize(op->s_d2h), "pcg batch");
    std::vector<PcgState> hs(static_cast<size_t>(nrhs));
    for (int k = 0; k < nrhs; ++k)
      ck(cudaMemcpy(&hs[size_t(k)], states + size_t(k) * sst, sizeof(PcgState),
                    cudaMemcpyDeviceToHost),
         "state");
    float tot = 0;
    ck(cudaEventElapsedTime(&tot, op->ev_t0, op->ev_t1), "elapsed");
    for (int k = 0; k < nrhs; ++k) {
      pcg_fill_report(op, hs[size_t(k)], hists + size_t(k) * hstride, launched[size_t(k)], false,
                      &reports[k]);
      reports[k].total_time_seconds = tot * 1e-3 / nrhs;  // batch wall share (device events)
    }
  });
}

}  // extern "C"
