/* hxf — C-ABI of the B200-native BP1-BP6 operator + PCG path.
 *
 * The drop-in boundary for the reference's (hexfem) operator API.  Plain
 * pointers and sizes only; every entry point returns an int status
 * (HXF_OK = 0) and leaves a thread-local message in hxf_last_error().  The
 * error classes map one to one onto the reference's exception types:
 *   HXF_EINVAL   <-> std::invalid_argument  (shape/size/parameter errors)
 *   HXF_ENUMERIC <-> std::runtime_error     (NaN, indefinite, det J <= 0)
 * (see proj/src/operator.cpp:26-46,67-68, pcg.cpp:27-31,54,75-91,
 *  qfunction.cpp:82-89,120 under /root/reference).
 *
 * Memory-space argument: HXF_HOST pointers are staged through pinned buffers
 * (functional parity with the reference's host-span signatures);
 * HXF_DEVICE pointers are used in place (the performance path).
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns HXF_ECUDA. */
#ifndef HXF_H
#define HXF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HXF_ABI_VERSION 2

typedef enum {
  HXF_OK = 0,
  HXF_EINVAL = 1,      /* std::invalid_argument */
  HXF_ENUMERIC = 2,    /* std::runtime_error (numerical failure) */
  HXF_ECUDA = 3,       /* CUDA runtime failure / no device */
  HXF_ENCCL = 4,       /* collective failure */
  HXF_EUNSUPPORTED = 5 /* (p, q, m) combination without a compiled kernel */
} hxf_status;

typedef enum { HXF_HOST = 0, HXF_DEVICE = 1 } hxf_memspace;
typedef enum { HXF_INTERP = 0, HXF_GRAD = 1 } hxf_eval_mode;          /* EvalMode */
typedef enum { HXF_FORWARD = 0, HXF_TRANSPOSE = 1 } hxf_eval_dir;      /* EvalDirection */
typedef enum { HXF_QDATA_MASS = 0, HXF_QDATA_DIFFUSION = 1 } hxf_qdata_kind; /* QDataKind */

typedef struct hxf_ctx hxf_ctx;
typedef struct hxf_op hxf_op;

/* Thread-local description of the last failure on this thread. */
const char* hxf_last_error(void);
int hxf_abi_version(void);
/* Number of hxf kernels launched so far in this process (instrumentation). */
int64_t hxf_launch_count(void);
/* Test knob: cap the grid of the operator and PCG vector kernels at `cap`
 * CTAs (0 = no cap; initial value from the HXF_MAX_GRID environment
 * variable), so small meshes exercise the multi-element-per-CTA loops the
 * full-size configurations run.  Returns the previous cap.  Affects launches
 * made (and graphs captured) after the call. */
int hxf_debug_set_grid_cap(int cap);
/* Test knob: operator-kernel family for the collocated fast paths (0: the
 * tuned dispatch — tensor-core kernels where available; 1: the register-line /
 * pencil kernels instead of the tensor-core ones; 2: the general kernel
 * op_apply_kernel everywhere, the A/B baseline and the path of bases that are
 * not centro-symmetric).  Initial value from HXF_OP_KERNEL; returns the
 * previous choice; affects launches made (and graphs captured) after the call. */
int hxf_debug_set_op_kernel(int choice);
/* Measurement knob: `on` != 0 makes the fused PCG step kernel record per-CTA
 * %globaltimer stamps (start, phase-1 end, after the grid barrier, phase-2
 * end) of its following launches; `out` (4 x 1024 uint64, or NULL) receives
 * the stamps of the last launch.  Current device. */
int hxf_debug_step_timestamps(int on, unsigned long long* out);

/* ---- context: one CUDA device (+ optional NCCL communicator) ----------- */
int hxf_context_create(int device, void* nccl_comm, hxf_ctx** out);
int hxf_context_destroy(hxf_ctx* ctx);
/* cudaStream_t the context launches on (as void*). */
void* hxf_context_stream(hxf_ctx* ctx);

/* ---- device memory on the context's device (stream-ordered on its stream) */
int hxf_malloc(hxf_ctx* ctx, uint64_t bytes, void** out);
int hxf_free(hxf_ctx* ctx, void* ptr);
/* kind: 0 host->device, 1 device->host, 2 device->device; synchronous. */
int hxf_memcpy(hxf_ctx* ctx, void* dst, const void* src, uint64_t bytes, int kind);
int hxf_synchronize(hxf_ctx* ctx);

/* ---- operator: replaces make_operator + MatFreeOperator --------------------
 * proj/include/hexfem/operator.hpp:19-38 (make_operator), validation as in
 * proj/src/operator.cpp:20-62.  Arrays are copied to the device at creation;
 * the handle is immutable afterwards. */
typedef struct {
  int p;                     /* basis degree (TensorBasis::p) */
  int q;                     /* 1-D quadrature points (TensorBasis::q) */
  int m;                     /* components (ElemRestriction::m) */
  int64_t num_elements;      /* ElemRestriction::num_elements */
  int64_t n_L;               /* ElemRestriction::n_L (scalar nodes) */
  const double* interp1d;    /* q x (p+1) row-major, TensorBasis::interp1d */
  const double* grad1d;      /* q x (p+1) row-major, TensorBasis::grad1d */
  const double* qpoints;     /* q quadrature points on [-1,1] (TensorBasis::quad.points) */
  const int64_t* indices;    /* num_elements x (p+1)^3, ElemRestriction::indices; NULL =
                                structured box given by dims (mesh.cpp:80-104 numbering) */
  int dims[3];               /* structured-box hint (elements per axis) or {0,0,0} */
  const double* mass_qdata;  /* E*q^3 (QData Mass values) or NULL */
  const double* diff_qdata;  /* E*6*q^3 (QData Diffusion values) or NULL */
  hxf_memspace qdata_space;  /* where the two qdata arrays live */
  double alpha, beta;        /* y = (alpha A + beta B) x */
  const int64_t* constrained;/* scalar L-indices (any order, duplicates allowed) */
  int64_t n_constrained;
  int block;                 /* KernelPlan::block — accepted and ignored */
} hxf_operator_desc;

int hxf_operator_create(hxf_ctx* ctx, const hxf_operator_desc* desc, hxf_op** out);
int hxf_operator_destroy(hxf_op* op);
/* size = m * n_L (MatFreeOperator::size) */
int64_t hxf_operator_size(const hxf_op* op);
/* 1 when the index table was recognised as the structured box and G/G^T are
 * computed from the lattice (no index traffic), 0 for the int32 table path. */
int hxf_operator_is_structured(const hxf_op* op);

/* operator_apply (operator.hpp:53-58, operator.cpp:64-144): y is overwritten;
 * constrained entries satisfy y = x.  stream: cudaStream_t or NULL for the
 * context stream.  Synchronous for HXF_HOST, stream-ordered for HXF_DEVICE. */
int hxf_operator_apply(hxf_op* op, const double* x, double* y, hxf_memspace space, void* stream);

/* operator_diagonal (operator.hpp:60-64, operator.cpp:170-256). */
int hxf_operator_diagonal(hxf_op* op, double* d, hxf_memspace space);

/* apply_g / apply_g_transpose over the operator's restriction
 * (restriction.hpp:35-42): E-vector layout e[(c*E+e)*S + s]. */
int hxf_restriction_apply(hxf_op* op, int transpose, const double* in, double* out,
                          hxf_memspace space);
/* multiplicity (restriction.hpp:44-45): n_L doubles. */
int hxf_restriction_multiplicity(hxf_op* op, double* out, hxf_memspace space);

/* apply_basis_batch (contraction.hpp:56-67, contraction.cpp:248-332) for ne
 * single-component element blocks; Grad data component-outermost across the
 * batch, (d*ne + e)*q^3.  Output overwritten. */
int hxf_basis_apply(hxf_ctx* ctx, int p, int q, const double* interp1d, const double* grad1d,
                    hxf_eval_mode mode, hxf_eval_dir dir, int64_t ne, const double* in,
                    double* out, hxf_memspace space);

/* apply_qf_mass / apply_qf_diffusion (qfunction.hpp:33-43) for elements
 * [e0, e0+ne) of a QData array of num_elements x (1|6) x nq values. */
int hxf_qfunction_apply(hxf_ctx* ctx, hxf_qdata_kind kind, const double* qdata,
                        int64_t num_elements, int nq, int64_t e0, int64_t ne, const double* in,
                        double* out, hxf_memspace space);

/* compute_qdata (qfunction.hpp:27-31, qfunction.cpp:12-122) on the device:
 * coords = 3*n_L component-major node coordinates, indices = E x (p+1)^3
 * (or NULL with dims set for the structured box), qweights = q 1-D weights.
 * out = E*(1|6)*q^3.  HXF_ENUMERIC when det J <= 0 (message names the
 * element and quadrature point). */
int hxf_qdata_compute(hxf_ctx* ctx, int p, int q, const double* interp1d, const double* grad1d,
                      const double* qweights, int64_t num_elements, int64_t n_L,
                      const double* coords, const int64_t* indices, const int dims[3],
                      hxf_qdata_kind kind, double* out, hxf_memspace space);

/* ---- standalone element restriction: replaces ElemRestriction ----------------
 * proj/include/hexfem/restriction.hpp:14-50 (make_restriction, apply_g,
 * apply_g_transpose, multiplicity, gather_scalar).  indices = E x (p+1)^3
 * int64 (verified entry by entry against the structured box, then not stored)
 * or NULL with dims set.  Lengths are the span sizes the reference checks;
 * a mismatch is HXF_EINVAL with the reference's message.  G^T accumulates in
 * the reference's colour-class order (bitwise equal) on the structured box. */
typedef struct hxf_restr hxf_restr;
int hxf_elem_restriction_create(hxf_ctx* ctx, int p, int m, int64_t num_elements, int64_t n_L,
                                const int64_t* indices, const int dims[3], hxf_restr** out);
int hxf_elem_restriction_destroy(hxf_restr* r);
int hxf_elem_restriction_is_structured(const hxf_restr* r);
/* transpose = 0: apply_g (in = m*n_L L-vector, out = m*E*S E-vector);
 * transpose = 1: apply_g_transpose (in = E-vector, out = L-vector, overwritten). */
int hxf_elem_restriction_apply(hxf_restr* r, int transpose, const double* in, int64_t in_len,
                               double* out, int64_t out_len, hxf_memspace space);
int hxf_elem_restriction_multiplicity(hxf_restr* r, double* out, int64_t out_len,
                                      hxf_memspace space);
/* gather_scalar (restriction.cpp:86-106): single-component G^T of E*S values. */
int hxf_elem_restriction_gather_scalar(hxf_restr* r, const double* e_scalar, int64_t e_len,
                                       double* l_scalar, int64_t l_len, hxf_memspace space);

/* ---- contraction kernels (contraction.hpp:43-75) ------------------------- */
/* contract_batch (contraction.cpp:177-206): the 1-D matrix (n_out x n_in
 * row-major, HOST) applied along tensor dimension dim of ne element blocks
 * of shape in_shape (x fastest); accumulate != 0 adds into out.  flops (or
 * NULL) is incremented by 2 per multiply-add like the reference's
 * FlopCounter.  Bitwise equal to the reference's sum-factorized path. */
int hxf_contract_batch(hxf_ctx* ctx, const double* matrix, int64_t matrix_len, int n_out,
                       int n_in, int dim, const int in_shape[3], int64_t ne, const double* in,
                       int64_t in_len, double* out, int64_t out_len, int accumulate,
                       hxf_memspace space, uint64_t* flops);
/* apply_tensor_3d (tensor_basis.hpp:38-47, tensor_basis.cpp:73-99): one
 * element, m components stored consecutively. */
int hxf_apply_tensor_3d(hxf_ctx* ctx, int p, int q, const double* interp1d, const double* grad1d,
                        hxf_eval_mode mode, hxf_eval_dir dir, int m, const double* u,
                        int64_t u_len, double* v, int64_t v_len, hxf_memspace space);
/* flops_estimate (contraction.cpp:334-340): multiply-adds x 2 per element of
 * the sum-factorized kernel; Grad = 3 x Interp; direction-independent. */
uint64_t hxf_flops_estimate(int p, int q, int m, hxf_eval_mode mode);

/* ---- structured-box setup on the device (build_mesh + bench.cpp fields) ----
 * The element box [off, off+loc) of a global box of glob elements (whole box:
 * off = 0, loc = glob), degree p, GLL nodes gll_nodes[p+1]: node coordinates
 * (3*n_L component-major, mesh.cpp:32-78 — bit-exact: the 1-D axes and their
 * sines are evaluated on the host as the reference does, the lattice and
 * sine bump on the device), and optionally the manufactured fields
 * (bench.cpp:56-62): u = sin(pi x) sin(pi y) sin(pi z) and f = 3 pi^2 u
 * (poisson) or u, each replicated over m components.  On the undeformed box
 * u and f are bit-exact too; on the sine box the deformed points' sines come
 * from the device's sin (within 1e-15 of max|u|).  Any of coords / f / u
 * may be NULL. */
int hxf_box_fields(hxf_ctx* ctx, const int glob[3], const int off[3], const int loc[3], int p,
                   const double* gll_nodes, int deform, int m, int poisson, double* coords,
                   double* f, double* u, hxf_memspace space);
/* v[c*n_L + i] = value on every constrained row i of the operator (device v). */
int hxf_operator_set_constrained(hxf_op* op, double* v, double value, hxf_memspace space);

/* ---- PCG: replaces pcg(ApplyFn, ...) for this operator ---------------------
 * proj/include/hexfem/pcg.hpp:13-41, proj/src/pcg.cpp:24-115.  x0 = 0;
 * diag = NULL means unpreconditioned.  Runs device-resident: only b (and the
 * diagonal) go in, x and the report come out. */
typedef struct {
  double tol_rel;       /* PcgOptions::tol_rel */
  int max_iter;         /* PcgOptions::max_iter */
  int fixed_iterations; /* PcgOptions::fixed_iterations, < 0 = unset */
  int time_apply;       /* 1: CUDA-event time every operator apply into
                           apply_time_seconds (the reference's timer,
                           pcg.cpp:70-73); costs ~7 us per apply inside the
                           fixed-iteration graph.  0: apply_time_seconds = 0 */
} hxf_pcg_options;

typedef struct {
  int iterations;            /* SolveReport::iterations */
  int converged;             /* SolveReport::converged */
  double* residual_history;  /* caller buffer, >= history_capacity entries; entry 0 = ||b|| */
  int history_capacity;
  double apply_time_seconds; /* device time inside the operator kernel (CUDA events) */
  double total_time_seconds; /* device time of the whole solve (CUDA events) */
} hxf_solve_report;

int hxf_pcg(hxf_op* op, const double* b, const double* diag, const hxf_pcg_options* opts,
            double* x, hxf_memspace space, hxf_solve_report* report);

/* nrhs consecutive solves with the same operator from HOST vectors b[k] into
 * x[k] (pinned memory for overlap), diag on the DEVICE (or NULL).  Pipelined
 * over three engines: the copy-in of b[k+1] and the copy-out of x[k-1] run
 * while solve k computes; each solve is exactly hxf_pcg's.  time_apply is
 * ignored (no per-apply events); reports[k].total_time_seconds is the batch's
 * device time / nrhs. */
int hxf_pcg_host_batch(hxf_op* op, int nrhs, const double* const* b, const double* diag,
                       const hxf_pcg_options* opts, double* const* x, hxf_solve_report* reports);

/* ---- partitioned box (multi-GPU) ---------------------------
 * The reference has no distributed layer (shared-memory threads only,
 * proj/src/parallel.cpp); this is the B200 extension its paper describes as
 * the gather-scatter P operator.  Each rank holds the
 * structured operator of one sub-box of the element grid; its L-vector is the
 * sub-box's own node lattice, interface planes duplicated.  A partitioned
 * operator's apply ends with an interface sum-exchange so every copy of an
 * interface node holds the assembled value; PCG dots weigh each node once
 * (owner = the sub-box in which it is not on a low interface plane) and are
 * all-reduced.  Restriction / basis / qfunction entry points stay local. */
typedef struct hxf_comm hxf_comm;
typedef struct hxf_comm_group hxf_comm_group;
#define HXF_COMM_ID_BYTES 128

/* NCCL (dlopen of libnccl.so.2): one rank per GPU.  Rank 0 makes the id and
 * distributes it (e.g. over torch.distributed); every rank then creates. */
int hxf_comm_unique_id(unsigned char id[HXF_COMM_ID_BYTES]);
int hxf_comm_create_nccl(hxf_ctx* ctx, int nranks, int rank, const unsigned char id[HXF_COMM_ID_BYTES],
                         hxf_comm** out);
/* Wrap a caller-owned ncclComm_t (not destroyed by hxf_comm_destroy). */
int hxf_comm_wrap_nccl(hxf_ctx* ctx, void* nccl_comm, hxf_comm** out);
/* In-process group: nranks sub-domains driven by nranks host threads (one
 * context each, any devices).  Host-synchronous, for tests and debugging. */
int hxf_comm_group_create(int nranks, hxf_comm_group** out);
int hxf_comm_group_destroy(hxf_comm_group* group);
int hxf_comm_create_group(hxf_ctx* ctx, hxf_comm_group* group, int rank, hxf_comm** out);
/* Peer-to-peer communicator: every rank stores its interface planes and dot
 * partials straight into the peers' mailboxes (NVLink peer stores between
 * GPUs, plain stores on one GPU) with system-scope flags; kernels only, so
 * CUDA-graph capturable.  Each rank allocates its mailbox (cap doubles per
 * interface plane, >= the largest m * plane) with hxf_comm_p2p_alloc, which
 * also returns its CUDA IPC handle; the caller gathers the handles (e.g. over
 * torch.distributed) and every rank then creates the communicator from the
 * nranks handles (bases may carry the pointers of mailboxes in this process;
 * NULL entries are opened from handles).  Ranks that share one process AND
 * device must not make device-synchronising calls (cudaFree, ...) while an
 * exchange is in flight: the receive kernels spin on the peers' flags. */
#define HXF_COMM_IPC_HANDLE_BYTES 64
int hxf_comm_p2p_alloc(hxf_ctx* ctx, int nranks, int64_t cap, void** base,
                       unsigned char handle[HXF_COMM_IPC_HANDLE_BYTES]);
int hxf_comm_create_p2p(hxf_ctx* ctx, int nranks, int rank, int64_t cap, void* const* bases,
                        const unsigned char* handles, hxf_comm** out);
/* Free a mailbox from hxf_comm_p2p_alloc (after every communicator using it is destroyed). */
int hxf_comm_p2p_free(hxf_ctx* ctx, void* base);
int hxf_comm_destroy(hxf_comm* comm);
int hxf_comm_rank(const hxf_comm* comm);
int hxf_comm_size(const hxf_comm* comm);
/* In-place sum over ranks of n doubles (device memory), on the stream (NULL = ctx stream). */
int hxf_comm_allreduce_sum(hxf_comm* comm, double* dev, int64_t n, void* stream);

typedef struct {
  int neighbor[3][2]; /* rank sharing this lattice's low / high face plane, per axis; -1 = none */
} hxf_partition_desc;
/* Attach a structured-box operator to a partition.  The constrained list
 * given at create time must already be the global-boundary faces only. */
int hxf_operator_set_partition(hxf_op* op, hxf_comm* comm, const hxf_partition_desc* desc);
/* Interface sum-exchange of an L-vector in place (the P^T P of the paper). */
int hxf_operator_halo_sum(hxf_op* op, double* v, hxf_memspace space);

#ifdef __cplusplus
}
#endif
#endif /* HXF_H */
