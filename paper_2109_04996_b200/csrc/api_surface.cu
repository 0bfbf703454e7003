// The rest of the reference's operator-level API surface on the C-ABI
// (include/hxf.h): a standalone element restriction (ElemRestriction with
// apply_g / apply_g_transpose / multiplicity / gather_scalar,
// restriction.hpp:33-50), contract_batch with its accumulate flag
// (contraction.hpp:51-54), apply_tensor_3d (tensor_basis.hpp:46-47) and the
// analytic flop count (flops_estimate, contraction.hpp:69-75).
//
// None of these is on the timed PCG path; they run the exact-order kernels of
// aux_kernels.cu, so their results are the reference's bit for bit (the
// restriction's G^T in the reference's colour-class order whenever the table
// is the structured box, which make_restriction always produces).
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "capi_internal.h"

struct hxf_restr {
  hxf_ctx* ctx = nullptr;
  int p = 0, m = 1, S = 0;
  int64_t E = 0, n_L = 0;
  bool structured = false;
  BoxDims box;
  int* d_idx = nullptr;  // int32 table when not the structured box
  Lattice lattice() const {
    Lattice L;
    L.p = p;
    L.S = S;
    L.E = E;
    L.n_L = n_L;
    L.NX = box.NX;
    L.NY = box.NY;
    L.nx = box.nx;
    L.ny = box.ny;
    L.nz = box.nz;
    return L;
  }
  ~hxf_restr() {
    if (d_idx) cudaFree(d_idx);
  }
};

namespace {

// Stage a host input (HXF_HOST) into a context scratch buffer.
const double* stage_in(DevVec& buf, const double* src, size_t n, hxf_memspace space,
                       cudaStream_t s) {
  if (space == HXF_DEVICE) return src;
  double* d = buf.ensure(n);
  if (n) h2d(d, src, n * 8, s);
  return d;
}

double* stage_out(DevVec& buf, double* dst, size_t n, hxf_memspace space) {
  return space == HXF_DEVICE ? dst : buf.ensure(n);
}

void finish_out(double* host, const double* dev, size_t n, hxf_memspace space, cudaStream_t s,
                const char* what) {
  if (space == HXF_HOST && n) d2h(host, dev, n * 8, s);
  ck(cudaStreamSynchronize(s), what);
}

}  // namespace

extern "C" {

int hxf_elem_restriction_create(hxf_ctx* ctx, int p, int m, int64_t num_elements, int64_t n_L,
                                const int64_t* indices, const int dims[3], hxf_restr** out) {
  return guarded([&] {
    if (!ctx || !out) fail(HXF_EINVAL, "make_restriction: NULL argument");
    if (m < 1) fail(HXF_EINVAL, "make_restriction: m must be >= 1");
    if (p < 1 || num_elements < 1 || n_L < 1)
      fail(HXF_EINVAL, "make_restriction: bad degree / element / node count");
    if (!indices && (!dims || dims[0] < 1 || dims[1] < 1 || dims[2] < 1))
      fail(HXF_EINVAL, "make_restriction: indices (or structured-box dims) are required");
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    auto r = std::make_unique<hxf_restr>();
    r->ctx = ctx;
    r->p = p;
    r->m = m;
    r->S = (p + 1) * (p + 1) * (p + 1);
    r->E = num_elements;
    r->n_L = n_L;
    if (indices)
      for (int64_t i = 0; i < num_elements * r->S; ++i)
        if (indices[i] < 0 || indices[i] >= n_L)
          fail(HXF_EINVAL, "make_restriction: restriction index out of range");
    r->structured = detect_box(p, num_elements, n_L, indices, dims, "make_restriction", &r->box);
    if (!r->structured) {
      if (n_L >= (int64_t(1) << 31)) fail(HXF_EUNSUPPORTED, "hxf: n_L >= 2^31 with a table");
      std::vector<int> idx32(size_t(num_elements * r->S));
      for (size_t i = 0; i < idx32.size(); ++i) idx32[i] = int(indices[i]);
      r->d_idx = dalloc<int>(idx32.size());
      ck(cudaMemcpy(r->d_idx, idx32.data(), idx32.size() * 4, cudaMemcpyHostToDevice),
         "index upload");
    }
    *out = r.release();
  });
}

int hxf_elem_restriction_destroy(hxf_restr* r) {
  return guarded([&] {
    if (!r) return;
    cudaStreamSynchronize(r->ctx->stream);
    delete r;
  });
}

int hxf_elem_restriction_is_structured(const hxf_restr* r) { return r && r->structured ? 1 : 0; }

int hxf_elem_restriction_apply(hxf_restr* r, int transpose, const double* in, int64_t in_len,
                               double* out, int64_t out_len, hxf_memspace space) {
  return guarded([&] {
    const char* who = transpose ? "apply_g_transpose" : "apply_g";
    if (!r || (!in && in_len) || (!out && out_len))
      fail(HXF_EINVAL, std::string(who) + ": NULL argument");
    const int64_t nl = int64_t(r->m) * r->n_L, ne = int64_t(r->m) * r->E * r->S;
    // restriction.cpp:31-34 / :53-56 (L-vector checked first)
    if ((transpose ? out_len : in_len) != nl)
      fail(HXF_EINVAL, std::string(who) + ": L-vector length mismatch");
    if ((transpose ? in_len : out_len) != ne)
      fail(HXF_EINVAL, std::string(who) + ": E-vector length mismatch");
    cudaStream_t s = r->ctx->stream;
    const double* din = stage_in(r->ctx->scratch_a, in, size_t(in_len), space, s);
    double* dout = stage_out(r->ctx->scratch_b, out, size_t(out_len), space);
    ck(launch_restriction(s, r->lattice(), r->d_idx, r->structured, r->m, transpose != 0, din,
                          dout),
       who);
    finish_out(out, dout, size_t(out_len), space, s, who);
  });
}

int hxf_elem_restriction_multiplicity(hxf_restr* r, double* out, int64_t out_len,
                                      hxf_memspace space) {
  return guarded([&] {
    if (!r || !out) fail(HXF_EINVAL, "multiplicity: NULL argument");
    if (out_len != r->n_L) fail(HXF_EINVAL, "multiplicity: L-vector length mismatch");
    cudaStream_t s = r->ctx->stream;
    double* dout = stage_out(r->ctx->scratch_b, out, size_t(out_len), space);
    ck(launch_multiplicity(s, r->lattice(), r->d_idx, dout), "multiplicity");
    finish_out(out, dout, size_t(out_len), space, s, "multiplicity");
  });
}

int hxf_elem_restriction_gather_scalar(hxf_restr* r, const double* e_scalar, int64_t e_len,
                                       double* l_scalar, int64_t l_len, hxf_memspace space) {
  return guarded([&] {
    if (!r || (!e_scalar && e_len) || !l_scalar)
      fail(HXF_EINVAL, "gather_scalar: NULL argument");
    // restriction.cpp:89-92
    if (l_len != r->n_L) fail(HXF_EINVAL, "gather_scalar: L-vector length mismatch");
    if (e_len != r->E * r->S) fail(HXF_EINVAL, "gather_scalar: E-vector length mismatch");
    cudaStream_t s = r->ctx->stream;
    const double* din = stage_in(r->ctx->scratch_a, e_scalar, size_t(e_len), space, s);
    double* dout = stage_out(r->ctx->scratch_b, l_scalar, size_t(l_len), space);
    ck(launch_restriction(s, r->lattice(), r->d_idx, r->structured, 1, true, din, dout),
       "gather_scalar");
    finish_out(l_scalar, dout, size_t(l_len), space, s, "gather_scalar");
  });
}

int hxf_contract_batch(hxf_ctx* ctx, const double* matrix, int64_t matrix_len, int n_out,
                       int n_in, int dim, const int in_shape[3], int64_t ne, const double* in,
                       int64_t in_len, double* out, int64_t out_len, int accumulate,
                       hxf_memspace space, uint64_t* flops) {
  return guarded([&] {
    if (!ctx || !in_shape || (!matrix && matrix_len) || (!in && in_len) || (!out && out_len))
      fail(HXF_EINVAL, "contract_batch: NULL argument");
    // contraction.cpp:181-189, same checks in the same order
    if (dim < 0 || dim > 2) fail(HXF_EINVAL, "contract_batch: dim must be 0, 1 or 2");
    if (n_out < 1 || n_in < 1 || in_shape[dim] != n_in)
      fail(HXF_EINVAL, "contract_batch: inconsistent shapes");
    if (matrix_len != int64_t(n_out) * n_in)
      fail(HXF_EINVAL, "contract_batch: matrix size mismatch");
    if (ne < 0 || in_shape[0] < 0 || in_shape[1] < 0 || in_shape[2] < 0)
      fail(HXF_EINVAL, "contract_batch: inconsistent shapes");
    const int64_t in_elem = int64_t(in_shape[0]) * in_shape[1] * in_shape[2];
    const int64_t out_elem = in_elem / n_in * n_out;
    if (in_len < ne * in_elem || out_len < ne * out_elem)
      fail(HXF_EINVAL, "contract_batch: buffer too small");
    cudaStream_t s = ctx->stream;
    double* dM = ctx->scratch_c.ensure(size_t(matrix_len));
    h2d(dM, matrix, size_t(matrix_len) * 8, s);
    const size_t nin = size_t(ne * in_elem), nout = size_t(ne * out_elem);
    const double* din = stage_in(ctx->scratch_a, in, nin, space, s);
    double* dout = space == HXF_DEVICE ? out : ctx->scratch_b.ensure(nout);
    if (space == HXF_HOST && accumulate && nout) h2d(dout, out, nout * 8, s);
    ck(launch_contract_batch(s, dM, n_out, n_in, dim, in_shape, ne, din, dout, accumulate != 0),
       "contract_batch");
    finish_out(out, dout, nout, space, s, "contract_batch");
    // FlopCounter semantics (contraction.cpp:171-173): 2 per multiply-add
    if (flops) *flops += 2 * uint64_t(ne) * uint64_t(out_elem) * uint64_t(n_in);
  });
}

int hxf_apply_tensor_3d(hxf_ctx* ctx, int p, int q, const double* interp1d, const double* grad1d,
                        hxf_eval_mode mode, hxf_eval_dir dir, int m, const double* u,
                        int64_t u_len, double* v, int64_t v_len, hxf_memspace space) {
  return guarded([&] {
    if (!ctx || !interp1d || !grad1d) fail(HXF_EINVAL, "apply_tensor_3d: NULL argument");
    // tensor_basis.cpp:75-88
    if (m < 1) fail(HXF_EINVAL, "apply_tensor_3d: m must be >= 1");
    if (p < 1 || q < 1 || p > 16 || q > 17) fail(HXF_EINVAL, "apply_tensor_3d: bad p/q");
    const int n1 = p + 1;
    const int64_t nd = int64_t(n1) * n1 * n1, nq = int64_t(q) * q * q;
    const bool fwd = dir == HXF_FORWARD, grad = mode == HXF_GRAD;
    const int64_t in_size = fwd ? nd : (grad ? 3 * nq : nq);
    const int64_t out_size = fwd ? (grad ? 3 * nq : nq) : nd;
    if (u_len != m * in_size || v_len != m * out_size || (!u && u_len) || (!v && v_len))
      fail(HXF_EINVAL, "apply_tensor_3d: shape mismatch");
    cudaStream_t s = ctx->stream;
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
    const double* du = stage_in(ctx->scratch_a, u, size_t(u_len), space, s);
    double* dv = stage_out(ctx->scratch_b, v, size_t(v_len), space);
    // components stored consecutively; each one is apply_basis_batch with
    // ne = 1 (tensor_basis.cpp:90-98)
    for (int c = 0; c < m; ++c)
      ck(launch_basis_apply(s, p, q, dt, dt + msz, dt + 2 * msz, dt + 3 * msz, int(mode), int(dir),
                            1, du + c * in_size, dv + c * out_size),
         "apply_tensor_3d");
    finish_out(v, dv, size_t(v_len), space, s, "apply_tensor_3d");
  });
}

int hxf_box_fields(hxf_ctx* ctx, const int glob[3], const int off[3], const int loc[3], int p,
                   const double* gll_nodes, int deform, int m, int poisson, double* coords,
                   double* f, double* u, hxf_memspace space) {
  return guarded([&] {
    if (!ctx || !glob || !off || !loc || !gll_nodes) fail(HXF_EINVAL, "build_mesh: NULL argument");
    if (p < 1) fail(HXF_EINVAL, "build_mesh: p must be >= 1");
    for (int a = 0; a < 3; ++a)
      if (glob[a] < 1 || loc[a] < 1 || off[a] < 0 || off[a] + loc[a] > glob[a])
        fail(HXF_EINVAL, "build_mesh: element counts must be >= 1");
    if (m < 1) fail(HXF_EINVAL, "bp_setup: m must be >= 1");
    cudaStream_t s = ctx->stream;
    // 1-D axes and their sines on the host, exactly as mesh.cpp:12-28,57-58
    // evaluate them (glibc sin): the only transcendental calls of the
    // undeformed fields
    int64_t gdim[3], ldim[3], noff[3];
    std::vector<double> axes;
    for (int a = 0; a < 3; ++a) {
      gdim[a] = int64_t(glob[a]) * p + 1;
      ldim[a] = int64_t(loc[a]) * p + 1;
      noff[a] = int64_t(off[a]) * p;
    }
    std::vector<double> c[3];
    for (int a = 0; a < 3; ++a) {
      const int ne = glob[a];
      c[a].assign(size_t(gdim[a]), 0.0);
      const double h = 1.0 / ne;
      for (int k = 0; k < ne; ++k)
        for (int j = 0; j <= p; ++j)
          c[a][size_t(k) * p + size_t(j)] = (k + 0.5 * (gll_nodes[j] + 1.0)) * h;
      c[a].back() = 1.0;
      c[a].front() = 0.0;
    }
    for (int a = 0; a < 3; ++a) axes.insert(axes.end(), c[a].begin(), c[a].end());
    for (int a = 0; a < 3; ++a)
      for (double v : c[a]) axes.push_back(std::sin(M_PI * v));
    const int64_t n_L = ldim[0] * ldim[1] * ldim[2];
    double* dax = ctx->scratch_c.ensure(axes.size());
    h2d(dax, axes.data(), axes.size() * 8, s);
    double* dc = coords;
    double* df = f;
    double* du = u;
    if (space == HXF_HOST) {  // staging: coords | f | u
      const size_t need = (coords ? 3 : 0) * size_t(n_L) + (f ? m : 0) * size_t(n_L) +
                          (u ? m : 0) * size_t(n_L);
      double* st = ctx->scratch_b.ensure(need);
      dc = coords ? st : nullptr;
      df = f ? st + (coords ? 3 * n_L : 0) : nullptr;
      du = u ? st + (coords ? 3 * n_L : 0) + (f ? int64_t(m) * n_L : 0) : nullptr;
    }
    ck(launch_box_fields(s, dax, gdim, noff, ldim, deform, m, poisson, dc, df, du), "box fields");
    if (space == HXF_HOST) {
      if (coords) d2h(coords, dc, size_t(3 * n_L) * 8, s);
      if (f) d2h(f, df, size_t(m) * n_L * 8, s);
      if (u) d2h(u, du, size_t(m) * n_L * 8, s);
    }
    ck(cudaStreamSynchronize(s), "box fields");
  });
}

int hxf_operator_set_constrained(hxf_op* op, double* v, double value, hxf_memspace space) {
  return guarded([&] {
    if (!op || !v) fail(HXF_EINVAL, "set_constrained: NULL argument");
    if (space != HXF_DEVICE) fail(HXF_EINVAL, "set_constrained: device vectors only");
    op_set_constrained(op, v, value, op->ctx->stream);
    ck(cudaStreamSynchronize(op->ctx->stream), "set_constrained");
  });
}

uint64_t hxf_flops_estimate(int p, int q, int m, hxf_eval_mode mode) {
  // contraction.cpp:334-340
  const uint64_t p1 = uint64_t(p) + 1, qq = uint64_t(q);
  const uint64_t interp = 2 * uint64_t(m) * (qq * p1 * p1 * p1 + qq * qq * p1 * p1 + qq * qq * qq * p1);
  return mode == HXF_INTERP ? interp : 3 * interp;
}

}  // extern "C"
