// Internal declarations shared by the hxf CUDA translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/hxf.h"

namespace hxf {

enum PcgError { PCG_OK = 0, PCG_ERR_RHS = 1, PCG_ERR_APPLY_NAN = 2, PCG_ERR_INDEFINITE = 3,
                PCG_ERR_RESID = 4 };

// Device-resident PCG scalars (pcg_kernels.cu, pcg_device.cuh).
// red[] holds this rank's reduction results; on a partitioned problem they
// are all-reduced in place between kernels ([0] pAp, [1] r.r, [2] r.z,
// [3] constrained p.p (owned rows), [4] b.b, [5] b.z).
struct PcgState {
  double red[8];
  double rho, pap, alpha, beta, norm_b, target, res, tol;
  double alpha_prev;  // alpha of the previous iteration (x updates batched in pairs)
  int it, stop, converged, error, limit, fixed;
  int stop_update;  // iteration whose update kernel stopped the solve (pAp check), 0 = none
  unsigned int counter[4];  // last-block counters: K1, update, direction, init
  unsigned int gbar[2];     // grid barrier of the fused update + direction kernel: count, generation
};

// Last-CTA finalisation of p.(A p) inside the operator kernel (PCG only):
// the CTA that finishes last sums every partial in a fixed order and derives
// alpha (pcg.cpp:74-82), so no separate reduction launch is needed.
struct PcgAlphaFin {
  PcgState* st;         // nullptr: plain apply
  const double* parts;  // all partials of this apply (earlier passes first)
  int nparts;           // partials written by earlier passes (this launch adds gridDim.x)
};

// Arguments of the fused operator kernel (op_kernel.cuh).
struct OpParams {
  const double* x;
  double* y;
  const double* qd;          // per-element padded geometric factors
  int64_t E, n_L;            // elements, scalar nodes (component stride)
  int64_t NX, NY, NZ;        // structured-box lattice
  int nx, ny;                // elements per axis (x, y)
  const int* idx;            // int32 E x P^3 table, or nullptr (structured box)
  int cons_mode;             // 0 none, 1 box faces (bnd_faces), 2 bitmask
  int bnd_faces;             // mode 1: bit 2d / 2d+1 = low / high face of axis d constrained
  const uint32_t* cons_mask; // n_L bits (mode 2)
  double* dot_partials;      // per-CTA partial of x_masked . y, or nullptr
  const int* stop;           // device flag: skip the whole kernel when set (PCG)
  double coef;               // alpha (diffusion) or beta (mass)
  int ablate;                // measurement-only ablation bits (HXF_ABLATE), 0 in production
  const double* D;           // device copy of the 1-D derivative matrix (collocated path)
  PcgAlphaFin fin;           // PCG: last-CTA alpha finalisation (fin.st == nullptr: off)
  int rev;                   // sweep elements last to first (L2 reuse across CG kernels)
  const int* elist;          // element ids to process (E entries), nullptr = 0..E-1 (DMMA kernel)
  int pdl;                   // launch with programmatic dependent launch (single apply)
  int cons_store;            // DMMA kernel: store y = x on the constrained rows it gathers
                             // (y zero-filled by the caller instead of preset by init_y)
};

// Is lattice node (ix, iy, iz) on a constrained face of the box (mode 1)?
__host__ __device__ inline bool on_bnd_face(const OpParams& p, int64_t ix, int64_t iy, int64_t iz) {
  const int f = p.bnd_faces;
  return (ix == 0 && (f & 1)) || (ix == p.NX - 1 && (f & 2)) || (iy == 0 && (f & 4)) ||
         (iy == p.NY - 1 && (f & 8)) || (iz == 0 && (f & 16)) || (iz == p.NZ - 1 && (f & 32));
}

// Launch the fused operator kernel instance for (P, Q, NC, interp, qk);
// returns cudaErrorNotSupported for an uninstantiated combination.
// B: q x p1 row-major interp1d, D: q x q derivative at the quadrature points.
cudaError_t launch_op(int P, int Q, int NC, bool interp, int qk, const OpParams& prm,
                      const double* B, const double* D, cudaStream_t s, int* grid_out);

// Upper bound on the grid of any launch_op() call (partials buffer size).
int max_op_grid();

// Test knob (hxf_debug_set_grid_cap / HXF_MAX_GRID): caps the grid of the
// operator and PCG vector kernels so small meshes run the multi-element-per-
// CTA (grid-stride) paths the full-size configurations take.  0 = no cap.
int grid_cap();
inline int capped_grid(int64_t want, int max_ctas) {
  int64_t g = want < max_ctas ? want : max_ctas;
  const int cap = grid_cap();
  if (cap > 0 && g > cap) g = cap;
  return (int)g;
}

// The even-odd line / pencil kernels need centro-symmetric 1-D matrices
// (B[q-1-i][p-j] = B[i][j], D[q-1-i][q-1-j] = -D[i][j]); otherwise the general
// kernel runs.
bool centro_symmetric(int P, int Q, bool interp, const double* B, const double* D);

// Per-P launchers (op_inst_p*.cu)
#define HXF_DECL_P(N)                                                                          \
  cudaError_t launch_op_p##N(int Q, int NC, bool interp, int qk, const OpParams& prm,       \
                             const double* B, const double* D, cudaStream_t s, int* grid_out);
HXF_DECL_P(2)
HXF_DECL_P(3)
HXF_DECL_P(4)
HXF_DECL_P(5)
HXF_DECL_P(6)
HXF_DECL_P(7)
HXF_DECL_P(8)
HXF_DECL_P(9)
HXF_DECL_P(10)
HXF_DECL_P(11)
HXF_DECL_P(12)
HXF_DECL_P(13)
HXF_DECL_P(14)
HXF_DECL_P(15)
HXF_DECL_P(16)
#undef HXF_DECL_P

int num_sms();

// Tensor map (CUtensorMap, 128 bytes) of an operator input viewed as the
// [m][NZ][NY][NX] f64 lattice with a 12x8x8x1 box (no swizzle), for
// the TMA gather of the structured-box kernels (encoded through the runtime's
// driver entry point; no libcuda link).  lattice_tma_ok: whether the lattice
// and pointer meet TMA's rules (16-byte aligned base, row / plane strides
// multiples of 16 bytes) and HXF_TMA is not 0.
bool lattice_tma_ok(const OpParams& prm, int m);
bool encode_lattice_map(const OpParams& prm, int m, void* map_out);
// HXF_OP_KERNEL selects the collocated fast path for A/B comparisons:
// unset/"dmma" -> 0 (tensor-core kernel where available), "pencil" -> 1,
// "generic" -> 2 (op_kernel.cuh only).
int op_kernel_choice();
bool pencil_disabled();
bool dmma_pad_disabled();
// HXF_DMMAEO: even-odd tensor-core kernel for P = p+1 = 9..16 (op_dmmaeo.cuh):
// unset / "1" where measured faster (P >= 13 one component, P >= 12 three),
// "2" every P = 9..16, "0" off
bool dmmaeo_enabled(int P, int ncomp);
bool step_ap_zero();
// HXF_DMMA3=0: BP6 p = 6, 7 on the component-by-component DMMA kernel instead
// of the component-batched one (op_dmma3.cuh)
bool dmma3_enabled();
bool step_pdl();
bool pdl_apply_disabled();    // HXF_PDL_APPLY=0: single apply without PDL (A/B)     // HXF_DMMA_PAD=0: p = 4..6 back on the pencil kernel (A/B)
bool pdl_enabled();           // HXF_PDL=1: programmatic dependent launch (off by default)
bool serpentine();            // HXF_SERPENTINE=0: all sweeps forward
int dmma_stages();
bool xbatch();  // PCG x updates batched over iteration pairs (HXF_XBATCH=0 disables)  // HXF_DMMA_STAGES: staged qdata buffers per CTA of op_dmma_kernel (1 default, 2)
int dmma_warps();  // HXF_DMMA_NW: warps per element of op_dmma_kernel (2, 4 default, 8)
int ablate_bits();
void count_launch(int n = 1);

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains; it must pdl_wait() before touching anything
// the predecessor writes.  Only for single-wave grids that also pdl_trigger().
template <class... KArgs, class... Args>
cudaError_t launch_pdl_if(bool allow, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = allow ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  return launch_pdl_if(pdl_enabled(), kern, grid, block, smem, s, std::forward<Args>(args)...);
}

}  // namespace hxf
