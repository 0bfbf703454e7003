/* TEST INFRASTRUCTURE ONLY — see hexfem_oracle.h.  CPU restatement of the
 * reference (hexfem) BP operator + PCG path.  Parity pinned against the
 * reference itself (oracle/_ref, tests/test_oracle_ref.py) and against the
 * golden vectors in tests/golden/ (tests/test_oracle_golden.py).
 *
 * Single threaded: the reference is bitwise independent of its pool size
 * (proj/include/hexfem/operator.hpp:53-55, parallel.hpp:13-16), so one worker
 * reproduces every pool size.  All citations are relative to
 * /root/reference/proj. */
#define _GNU_SOURCE
#include "hexfem_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }
const char* orc_impl_name(void) { return "oracle-c"; }

/* ------------------------------------------------------------------ quadrature
 * Newton on Legendre polynomials, lower half mirrored (src/quadrature.cpp:17-126). */
static void legendre(int n, double x, double* val, double* der) {
  if (n == 0) { *val = 1.0; *der = 0.0; return; }
  double pm1 = 1.0, p = x;
  for (int k = 1; k < n; ++k) {
    const double pk1 = ((2 * k + 1) * x * p - k * pm1) / (k + 1);
    pm1 = p;
    p = pk1;
  }
  const double denom = x * x - 1.0;
  double dp;
  if (fabs(denom) > 1e-10)
    dp = n * (x * p - pm1) / denom;
  else
    dp = 0.5 * n * (n + 1) * (x >= 0 ? 1.0 : (n % 2 ? 1.0 : -1.0));
  *val = p;
  *der = dp;
}

int orc_quadrature(int kind, int q, double* pts, double* wts) {
  double p, dp;
  if (kind == 0) {
    if (q < 1) return fail(1, "make_quadrature: Gauss-Legendre needs q >= 1");
    for (int i = 0; i < q / 2; ++i) {
      double x = -cos(M_PI * (i + 0.75) / (q + 0.5));
      for (int it = 0; it < 100; ++it) {
        legendre(q, x, &p, &dp);
        const double dx = p / dp;
        x -= dx;
        if (fabs(dx) <= 1e-15) break;
      }
      legendre(q, x, &p, &dp);
      const double w = 2.0 / ((1.0 - x * x) * dp * dp);
      pts[i] = x;
      wts[i] = w;
      pts[q - 1 - i] = -x;
      wts[q - 1 - i] = w;
    }
    if (q % 2 == 1) {
      legendre(q, 0.0, &p, &dp);
      pts[q / 2] = 0.0;
      wts[q / 2] = 2.0 / (dp * dp);
    }
    return 0;
  }
  if (q < 2) return fail(1, "make_quadrature: Gauss-Lobatto-Legendre needs q >= 2");
  const int n = q - 1;
  const double end_w = 2.0 / ((double)n * (n + 1));
  pts[0] = -1.0;
  pts[q - 1] = 1.0;
  wts[0] = end_w;
  wts[q - 1] = end_w;
  for (int i = 1; i < q / 2; ++i) {
    double x = -cos(M_PI * i / n);
    for (int it = 0; it < 100; ++it) {
      legendre(n, x, &p, &dp);
      const double d2p = (2.0 * x * dp - (double)n * (n + 1) * p) / (1.0 - x * x);
      const double dx = dp / d2p;
      x -= dx;
      if (fabs(dx) <= 1e-15) break;
    }
    legendre(n, x, &p, &dp);
    const double w = 2.0 / ((double)n * (n + 1) * p * p);
    pts[i] = x;
    wts[i] = w;
    pts[q - 1 - i] = -x;
    wts[q - 1 - i] = w;
  }
  if (q % 2 == 1) {
    legendre(n, 0.0, &p, &dp);
    pts[q / 2] = 0.0;
    wts[q / 2] = 2.0 / ((double)n * (n + 1) * p * p);
  }
  return 0;
}

/* ------------------------------------------------------------------ basis
 * Lagrange basis on p+1 GLL nodes tabulated at the rule (src/tensor_basis.cpp:10-71). */
typedef struct {
  int p, q, kind, collocated;
  double *nodes, *qpts, *qwts;
  double *B, *G, *Bt, *Gt; /* q x (p+1) row-major, and (p+1) x q */
} Basis;

static double lag_val(const double* nd, int n, int j, double x) {
  double r = 1.0;
  for (int m = 0; m < n; ++m)
    if (m != j) r *= (x - nd[m]) / (nd[j] - nd[m]);
  return r;
}

static double lag_der(const double* nd, int n, int j, double x) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    if (i == j) continue;
    double prod = 1.0;
    for (int m = 0; m < n; ++m)
      if (m != i && m != j) prod *= (x - nd[m]) / (nd[j] - nd[m]);
    s += prod / (nd[j] - nd[i]);
  }
  return s;
}

static void basis_free(Basis* b) {
  free(b->nodes); free(b->qpts); free(b->qwts);
  free(b->B); free(b->G); free(b->Bt); free(b->Gt);
  memset(b, 0, sizeof *b);
}

static int basis_make(Basis* b, int p, int kind, int q) {
  memset(b, 0, sizeof *b);
  if (p < 1) return fail(1, "make_basis: p must be >= 1");
  const int n1 = p + 1;
  b->p = p; b->q = q; b->kind = kind;
  b->nodes = malloc(sizeof(double) * n1);
  double* tmpw = malloc(sizeof(double) * n1);
  b->qpts = malloc(sizeof(double) * q);
  b->qwts = malloc(sizeof(double) * q);
  int rc = orc_quadrature(1, n1, b->nodes, tmpw);
  free(tmpw);
  if (rc == 0) rc = orc_quadrature(kind, q, b->qpts, b->qwts);
  if (rc) { basis_free(b); return rc; }
  b->collocated = (kind == 1 && q == n1);
  b->B = malloc(sizeof(double) * q * n1);
  b->G = malloc(sizeof(double) * q * n1);
  b->Bt = malloc(sizeof(double) * q * n1);
  b->Gt = malloc(sizeof(double) * q * n1);
  for (int iq = 0; iq < q; ++iq)
    for (int j = 0; j < n1; ++j) {
      b->B[iq * n1 + j] = lag_val(b->nodes, n1, j, b->qpts[iq]);
      b->G[iq * n1 + j] = lag_der(b->nodes, n1, j, b->qpts[iq]);
    }
  for (int iq = 0; iq < q; ++iq)
    for (int j = 0; j < n1; ++j) {
      b->Bt[j * q + iq] = b->B[iq * n1 + j];
      b->Gt[j * q + iq] = b->G[iq * n1 + j];
    }
  return 0;
}

int orc_basis(int p, int kind, int q, double* interp, double* grad) {
  Basis b;
  int rc = basis_make(&b, p, kind, q);
  if (rc) return rc;
  memcpy(interp, b.B, sizeof(double) * q * (p + 1));
  memcpy(grad, b.G, sizeof(double) * q * (p + 1));
  basis_free(&b);
  return 0;
}

/* ------------------------------------------------------------------ contraction
 * One 1D contraction along `dim`, contracted index innermost and increasing
 * (src/contraction.cpp:14-76).  s = input shape (x fastest). */
static void contract(const double* M, int n_out, int n_in, int dim, const int s[3],
                     const double* in, double* out, int accumulate) {
  if (dim == 0) {
    for (int c = 0; c < s[2]; ++c)
      for (int b = 0; b < s[1]; ++b) {
        const double* col = in + (int64_t)n_in * (b + (int64_t)s[1] * c);
        double* orow = out + (int64_t)n_out * (b + (int64_t)s[1] * c);
        for (int a1 = 0; a1 < n_out; ++a1) {
          const double* row = M + (int64_t)a1 * n_in;
          double acc = 0.0;
          for (int a = 0; a < n_in; ++a) acc += row[a] * col[a];
          if (accumulate) orow[a1] += acc; else orow[a1] = acc;
        }
      }
  } else if (dim == 1) {
    for (int c = 0; c < s[2]; ++c)
      for (int b1 = 0; b1 < n_out; ++b1) {
        const double* row = M + (int64_t)b1 * n_in;
        for (int a = 0; a < s[0]; ++a) {
          double acc = 0.0;
          for (int b = 0; b < n_in; ++b)
            acc += row[b] * in[a + (int64_t)s[0] * (b + (int64_t)s[1] * c)];
          double* o = &out[a + (int64_t)s[0] * (b1 + (int64_t)n_out * c)];
          if (accumulate) *o += acc; else *o = acc;
        }
      }
  } else {
    const int64_t plane = (int64_t)s[0] * s[1];
    for (int c1 = 0; c1 < n_out; ++c1) {
      const double* row = M + (int64_t)c1 * n_in;
      for (int b = 0; b < s[1]; ++b)
        for (int a = 0; a < s[0]; ++a) {
          double acc = 0.0;
          for (int c = 0; c < n_in; ++c) acc += row[c] * in[a + (int64_t)s[0] * b + plane * c];
          double* o = &out[a + (int64_t)s[0] * b + plane * c1];
          if (accumulate) *o += acc; else *o = acc;
        }
    }
  }
}

/* Three-stage chain, forward dims 0,1,2 / transpose dims 2,1,0, for ONE
 * element (src/contraction.cpp:212-238).  Per-element arithmetic does not
 * depend on the batch size, so element-at-a-time reproduces any batching. */
static void chain3(const double* m0, const double* m1, const double* m2, int nn, int nq,
                   int transpose, const double* in, double* out, double* ta, double* tb,
                   int acc_last) {
  int s[3];
  if (!transpose) {
    s[0] = nn; s[1] = nn; s[2] = nn;
    contract(m0, nq, nn, 0, s, in, ta, 0);
    s[0] = nq;
    contract(m1, nq, nn, 1, s, ta, tb, 0);
    s[1] = nq;
    contract(m2, nq, nn, 2, s, tb, out, acc_last);
  } else {
    s[0] = nq; s[1] = nq; s[2] = nq;
    contract(m2, nn, nq, 2, s, in, ta, 0);
    s[2] = nn;
    contract(m1, nn, nq, 1, s, ta, tb, 0);
    s[1] = nn;
    contract(m0, nn, nq, 0, s, tb, out, acc_last);
  }
}

/* apply_basis_batch sum-factorized path (src/contraction.cpp:248-295): Grad
 * data is component-outermost across the batch, (d*ne + e)*q^3. */
static void basis_batch(const Basis* b, int grad, int transpose, int64_t ne, const double* in,
                        double* out, double* ta, double* tb) {
  const int nn = b->p + 1, nq = b->q;
  const int64_t nd3 = (int64_t)nn * nn * nn, nq3 = (int64_t)nq * nq * nq;
  for (int64_t e = 0; e < ne; ++e) {
    if (!grad) {
      if (!transpose)
        chain3(b->B, b->B, b->B, nn, nq, 0, in + e * nd3, out + e * nq3, ta, tb, 0);
      else
        chain3(b->Bt, b->Bt, b->Bt, nn, nq, 1, in + e * nq3, out + e * nd3, ta, tb, 0);
      continue;
    }
    for (int d = 0; d < 3; ++d) {
      const double* f[3] = {b->B, b->B, b->B};
      const double* ft[3] = {b->Bt, b->Bt, b->Bt};
      f[d] = b->G;
      ft[d] = b->Gt;
      if (!transpose)
        chain3(f[0], f[1], f[2], nn, nq, 0, in + e * nd3, out + (d * ne + e) * nq3, ta, tb, 0);
      else
        chain3(ft[0], ft[1], ft[2], nn, nq, 1, in + (d * ne + e) * nq3, out + e * nd3, ta, tb,
               d > 0);
    }
  }
}

int orc_apply_basis(int p, int kind, int q, int mode, int dir, int64_t ne, const double* in,
                    int64_t n_in, double* out, int64_t n_out) {
  Basis b;
  int rc = basis_make(&b, p, kind, q);
  if (rc) return rc;
  const int64_t nd3 = (int64_t)(p + 1) * (p + 1) * (p + 1), nq3 = (int64_t)q * q * q;
  const int64_t in_e = (mode && dir) ? 3 * nq3 : (!dir ? nd3 : nq3);
  const int64_t out_e = (mode && !dir) ? 3 * nq3 : (!dir ? nq3 : nd3);
  if (n_in < ne * in_e || n_out < ne * out_e) {
    basis_free(&b);
    return fail(1, "apply_basis_batch: buffer too small");
  }
  const int mx = (p + 1) > q ? p + 1 : q;
  double* ta = malloc(sizeof(double) * mx * mx * mx);
  double* tb = malloc(sizeof(double) * mx * mx * mx);
  basis_batch(&b, mode, dir, ne, in, out, ta, tb);
  free(ta); free(tb);
  basis_free(&b);
  return 0;
}

/* contract_batch (src/contraction.cpp:177-206): the same checks in the same
 * order, then contract_sf element by element; 2 flops per multiply-add. */
int orc_contract_batch(const double* M, int64_t m_len, int n_out, int n_in, int dim,
                       const int* shape, int64_t ne, const double* in, int64_t in_len, double* out,
                       int64_t out_len, int accumulate, uint64_t* flops) {
  if (dim < 0 || dim > 2) return fail(1, "contract_batch: dim must be 0, 1 or 2");
  if (n_out < 1 || n_in < 1 || shape[dim] != n_in)
    return fail(1, "contract_batch: inconsistent shapes");
  if (m_len != (int64_t)n_out * n_in) return fail(1, "contract_batch: matrix size mismatch");
  const int64_t in_elem = (int64_t)shape[0] * shape[1] * shape[2];
  const int64_t out_elem = in_elem / n_in * n_out;
  if (in_len < ne * in_elem || out_len < ne * out_elem)
    return fail(1, "contract_batch: buffer too small");
  for (int64_t e = 0; e < ne; ++e)
    contract(M, n_out, n_in, dim, shape, in + e * in_elem, out + e * out_elem, accumulate);
  if (flops) *flops += 2 * (uint64_t)ne * (uint64_t)out_elem * (uint64_t)n_in;
  return 0;
}

/* apply_tensor_3d (src/tensor_basis.cpp:73-99): m components stored
 * consecutively, each an apply_basis_batch with ne = 1. */
int orc_apply_tensor_3d(int p, int kind, int q, int mode, int dir, int m, const double* u,
                        int64_t u_len, double* v, int64_t v_len) {
  if (m < 1) return fail(1, "apply_tensor_3d: m must be >= 1");
  Basis b;
  int rc = basis_make(&b, p, kind, q);
  if (rc) return rc;
  const int64_t nd = (int64_t)(p + 1) * (p + 1) * (p + 1), nq = (int64_t)q * q * q;
  const int64_t in_size = !dir ? nd : (mode ? 3 * nq : nq);
  const int64_t out_size = !dir ? (mode ? 3 * nq : nq) : nd;
  if (u_len != m * in_size || v_len != m * out_size) {
    basis_free(&b);
    return fail(1, "apply_tensor_3d: shape mismatch");
  }
  const int mx = (p + 1) > q ? p + 1 : q;
  double* ta = malloc(sizeof(double) * mx * mx * mx);
  double* tb = malloc(sizeof(double) * mx * mx * mx);
  for (int c = 0; c < m; ++c) basis_batch(&b, mode, dir, 1, u + c * in_size, v + c * out_size, ta, tb);
  free(ta); free(tb);
  basis_free(&b);
  return 0;
}

/* flops_estimate (src/contraction.cpp:334-340) */
uint64_t orc_flops_estimate(int p, int q, int m, int mode) {
  const uint64_t p1 = (uint64_t)p + 1, qq = (uint64_t)q;
  const uint64_t interp = 2 * (uint64_t)m * (qq * p1 * p1 * p1 + qq * qq * p1 * p1 + qq * qq * qq * p1);
  return mode ? 3 * interp : interp;
}

/* apply_basis_batch with a counter: chain3's three contractions per chain,
 * counted like contract_sf<true> (one per multiply-add, 2 flops each). */
int orc_apply_basis_counted(int p, int kind, int q, int mode, int dir, int64_t ne,
                            const double* in, int64_t n_in, double* out, int64_t n_out,
                            uint64_t* flops) {
  const int rc = orc_apply_basis(p, kind, q, mode, dir, ne, in, n_in, out, n_out);
  if (rc) return rc;
  const uint64_t n1 = (uint64_t)p + 1, qq = (uint64_t)q;
  const uint64_t chain = qq * n1 * n1 * n1 + qq * qq * n1 * n1 + qq * qq * qq * n1;
  if (flops) *flops += 2 * (uint64_t)ne * chain * (mode ? 3 : 1);
  return 0;
}

/* ------------------------------------------------------------------ mesh
 * Structured unit-cube hex mesh, GLL lattice, optional sine bump
 * (src/mesh.cpp:12-78); element node indices (src/mesh.cpp:80-104). */
typedef struct {
  int dims[3], p;
  int64_t NX, NY, NZ, n_L, E;
  double* coords; /* 3*n_L component-major */
  int64_t* boundary;
  int64_t n_boundary;
} Mesh;

static double* axis_coords(int nx, int p) {
  double* gll = malloc(sizeof(double) * (p + 1));
  double* w = malloc(sizeof(double) * (p + 1));
  orc_quadrature(1, p + 1, gll, w);
  const int64_t n = (int64_t)nx * p + 1;
  double* c = malloc(sizeof(double) * n);
  const double h = 1.0 / nx;
  for (int k = 0; k < nx; ++k)
    for (int j = 0; j <= p; ++j) c[(int64_t)k * p + j] = (k + 0.5 * (gll[j] + 1.0)) * h;
  c[n - 1] = 1.0;
  c[0] = 0.0;
  free(gll); free(w);
  return c;
}

static void mesh_build(Mesh* m, int nx, int ny, int nz, int p, int sine) {
  memset(m, 0, sizeof *m);
  m->dims[0] = nx; m->dims[1] = ny; m->dims[2] = nz; m->p = p;
  m->NX = (int64_t)nx * p + 1; m->NY = (int64_t)ny * p + 1; m->NZ = (int64_t)nz * p + 1;
  m->n_L = m->NX * m->NY * m->NZ;
  m->E = (int64_t)nx * ny * nz;
  m->coords = malloc(sizeof(double) * 3 * m->n_L);
  m->boundary = malloc(sizeof(int64_t) * m->n_L);
  double* cx = axis_coords(nx, p);
  double* cy = axis_coords(ny, p);
  double* cz = axis_coords(nz, p);
  int64_t node = 0;
  for (int64_t iz = 0; iz < m->NZ; ++iz)
    for (int64_t iy = 0; iy < m->NY; ++iy)
      for (int64_t ix = 0; ix < m->NX; ++ix, ++node) {
        double x = cx[ix], y = cy[iy], z = cz[iz];
        if (sine) {
          const double bump = 0.05 * sin(M_PI * x) * sin(M_PI * y) * sin(M_PI * z);
          x += bump; y += bump; z += bump;
        }
        m->coords[node] = x;
        m->coords[m->n_L + node] = y;
        m->coords[2 * m->n_L + node] = z;
        if (ix == 0 || ix == m->NX - 1 || iy == 0 || iy == m->NY - 1 || iz == 0 ||
            iz == m->NZ - 1)
          m->boundary[m->n_boundary++] = node;
      }
  free(cx); free(cy); free(cz);
}

static void mesh_free(Mesh* m) { free(m->coords); free(m->boundary); }

/* ------------------------------------------------------------------ restriction
 * Index table + 8 parity colours (src/restriction.cpp:7-26). */
typedef struct {
  int64_t E, n_L;
  int S, m;
  int64_t* idx;      /* E*S */
  int64_t* color_el; /* E, grouped by colour */
  int64_t color_off[9];
} Restr;

static void restr_make(Restr* r, const Mesh* mesh, int m) {
  const int p = mesh->p, n1 = p + 1;
  r->E = mesh->E; r->n_L = mesh->n_L; r->S = n1 * n1 * n1; r->m = m;
  r->idx = malloc(sizeof(int64_t) * r->E * r->S);
  r->color_el = malloc(sizeof(int64_t) * r->E);
  int64_t count[8] = {0};
  for (int64_t e = 0; e < r->E; ++e) {
    const int64_t ex = e % mesh->dims[0];
    const int64_t ey = (e / mesh->dims[0]) % mesh->dims[1];
    const int64_t ez = e / ((int64_t)mesh->dims[0] * mesh->dims[1]);
    int64_t* out = r->idx + e * r->S;
    int s = 0;
    for (int kz = 0; kz <= p; ++kz)
      for (int ky = 0; ky <= p; ++ky)
        for (int kx = 0; kx <= p; ++kx)
          out[s++] = (ex * p + kx) + mesh->NX * ((ey * p + ky) + mesh->NY * (ez * p + kz));
    count[(ex & 1) | ((ey & 1) << 1) | ((ez & 1) << 2)]++;
  }
  r->color_off[0] = 0;
  for (int c = 0; c < 8; ++c) r->color_off[c + 1] = r->color_off[c] + count[c];
  int64_t fill[8];
  for (int c = 0; c < 8; ++c) fill[c] = r->color_off[c];
  for (int64_t e = 0; e < r->E; ++e) {
    const int64_t ex = e % mesh->dims[0];
    const int64_t ey = (e / mesh->dims[0]) % mesh->dims[1];
    const int64_t ez = e / ((int64_t)mesh->dims[0] * mesh->dims[1]);
    r->color_el[fill[(ex & 1) | ((ey & 1) << 1) | ((ez & 1) << 2)]++] = e;
  }
}

static void restr_free(Restr* r) { free(r->idx); free(r->color_el); }

/* apply_g: pure copy L -> E (src/restriction.cpp:28-48). */
static void apply_g(const Restr* r, const double* l, double* ev) {
  for (int c = 0; c < r->m; ++c)
    for (int64_t e = 0; e < r->E; ++e) {
      const int64_t* idx = r->idx + e * r->S;
      double* out = ev + (c * r->E + e) * r->S;
      for (int s = 0; s < r->S; ++s) out[s] = l[c * r->n_L + idx[s]];
    }
}

/* apply_g_transpose: zero, then colour classes in increasing id
 * (src/restriction.cpp:50-75).  `ncomp` = 1 gives gather_scalar (:86-106). */
static void apply_gt(const Restr* r, int ncomp, const double* ev, double* l) {
  memset(l, 0, sizeof(double) * ncomp * r->n_L);
  for (int col = 0; col < 8; ++col)
    for (int c = 0; c < ncomp; ++c)
      for (int64_t k = r->color_off[col]; k < r->color_off[col + 1]; ++k) {
        const int64_t e = r->color_el[k];
        const int64_t* idx = r->idx + e * r->S;
        const double* in = ev + (c * r->E + e) * r->S;
        for (int s = 0; s < r->S; ++s) l[c * r->n_L + idx[s]] += in[s];
      }
}

/* ------------------------------------------------------------------ qdata
 * Geometric factors (src/qfunction.cpp:12-122).  kind 0 mass w*det,
 * 1 diffusion upper triangle of w*det*J^-1 J^-T at ((e*6+s)*nq + qi). */
static int qdata_compute(const Mesh* mesh, const Basis* b, int kind, double** out_vals) {
  const int64_t E = mesh->E;
  const int q = b->q, nq = q * q * q, nn = b->p + 1, S = nn * nn * nn;
  const int K = kind == 0 ? 1 : 6;
  double* vals = calloc((size_t)E * K * nq, sizeof(double));
  double* wq = malloc(sizeof(double) * nq);
  for (int c = 0, i = 0; c < q; ++c)
    for (int bb = 0; bb < q; ++bb)
      for (int a = 0; a < q; ++a, ++i) wq[i] = b->qwts[a] * b->qwts[bb] * b->qwts[c];
  Restr r3;
  restr_make(&r3, mesh, 3);
  double* ec = malloc(sizeof(double) * 3 * E * S);
  apply_g(&r3, mesh->coords, ec);
  const int mx = nn > q ? nn : q;
  double* ta = malloc(sizeof(double) * mx * mx * mx);
  double* tb = malloc(sizeof(double) * mx * mx * mx);
  double* grad = malloc(sizeof(double) * 9 * nq);
  int rc = 0;
  for (int64_t e = 0; e < E && !rc; ++e) {
    for (int a = 0; a < 3; ++a)
      basis_batch(b, 1, 0, 1, ec + (a * E + e) * S, grad + a * 3 * nq, ta, tb);
    for (int qi = 0; qi < nq; ++qi) {
      double J[3][3];
      for (int a = 0; a < 3; ++a)
        for (int d = 0; d < 3; ++d) J[a][d] = grad[(a * 3 + d) * nq + qi];
      const double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1]) -
                         J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0]) +
                         J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
      if (!(det > 0.0)) {
        snprintf(g_err, sizeof g_err,
                 "compute_qdata: non-positive Jacobian determinant (%f) in element %lld at "
                 "quadrature point %d", det, (long long)e, qi);
        rc = 2;
        break;
      }
      const double wdet = wq[qi] * det;
      if (kind == 0) {
        vals[e * nq + qi] = wdet;
        continue;
      }
      double inv[3][3];
      inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
      inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
      inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
      inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
      int s = 0;
      for (int a = 0; a < 3; ++a)
        for (int bb = a; bb < 3; ++bb, ++s) {
          const double v = inv[a][0] * inv[bb][0] + inv[a][1] * inv[bb][1] + inv[a][2] * inv[bb][2];
          vals[(e * 6 + s) * nq + qi] = wdet * v;
        }
    }
  }
  free(wq); free(ec); free(ta); free(tb); free(grad);
  restr_free(&r3);
  if (rc) { free(vals); return rc; }
  *out_vals = vals;
  return 0;
}

/* ------------------------------------------------------------------ operator */
typedef struct {
  Restr r;
  const Basis* basis;
  const double* mass_qd; /* E*nq or NULL */
  const double* diff_qd; /* E*6*nq or NULL */
  int m;
  double alpha, beta;
  const int64_t* cons;
  int64_t ncons;
} Op;

/* operator_apply (src/operator.cpp:64-144): mask -> G -> per element
 * B, D, B^T -> colour-ordered G^T -> y += coef*l -> constrained identity. */
static void op_apply(const Op* op, const double* x, double* y) {
  const Restr* r = &op->r;
  const int64_t E = r->E, S = r->S, n_L = r->n_L, n = (int64_t)op->m * n_L;
  const Basis* b = op->basis;
  const int q = b->q, nq = q * q * q, nn = b->p + 1;
  const int mx = nn > q ? nn : q;
  double* masked = malloc(sizeof(double) * n);
  double* ein = malloc(sizeof(double) * op->m * E * S);
  double* eout = malloc(sizeof(double) * op->m * E * S);
  double* ltmp = malloc(sizeof(double) * n);
  double* qin = malloc(sizeof(double) * 3 * nq);
  double* qout = malloc(sizeof(double) * 3 * nq);
  double* ta = malloc(sizeof(double) * mx * mx * mx);
  double* tb = malloc(sizeof(double) * mx * mx * mx);
  memcpy(masked, x, sizeof(double) * n);
  for (int c = 0; c < op->m; ++c)
    for (int64_t k = 0; k < op->ncons; ++k) masked[c * n_L + op->cons[k]] = 0.0;
  for (int64_t i = 0; i < n; ++i) y[i] = 0.0;
  for (int stage = 0; stage < 2; ++stage) {
    const int grad = stage == 0;
    const double coef = grad ? op->alpha : op->beta;
    if (coef == 0.0) continue;
    apply_g(r, masked, ein);
    for (int64_t e = 0; e < E; ++e)
      for (int c = 0; c < op->m; ++c) {
        const double* in = ein + (c * E + e) * S;
        double* out = eout + (c * E + e) * S;
        basis_batch(b, grad, 0, 1, in, qin, ta, tb);
        if (grad) {
          /* apply_qf_diffusion (src/qfunction.cpp:135-162) */
          const double* s = op->diff_qd + e * 6 * nq;
          for (int i = 0; i < nq; ++i) {
            const double u0 = qin[i], u1 = qin[nq + i], u2 = qin[2 * nq + i];
            qout[i] = s[i] * u0 + s[nq + i] * u1 + s[2 * nq + i] * u2;
            qout[nq + i] = s[nq + i] * u0 + s[3 * nq + i] * u1 + s[4 * nq + i] * u2;
            qout[2 * nq + i] = s[2 * nq + i] * u0 + s[4 * nq + i] * u1 + s[5 * nq + i] * u2;
          }
        } else {
          /* apply_qf_mass (src/qfunction.cpp:124-133) */
          const double* w = op->mass_qd + e * nq;
          for (int i = 0; i < nq; ++i) qout[i] = w[i] * qin[i];
        }
        basis_batch(b, grad, 1, 1, qout, out, ta, tb);
      }
    apply_gt(r, op->m, eout, ltmp);
    for (int64_t i = 0; i < n; ++i) y[i] += coef * ltmp[i];
  }
  for (int c = 0; c < op->m; ++c)
    for (int64_t k = 0; k < op->ncons; ++k) y[c * n_L + op->cons[k]] = x[c * n_L + op->cons[k]];
  free(masked); free(ein); free(eout); free(ltmp); free(qin); free(qout); free(ta); free(tb);
}

/* operator_diagonal (src/operator.cpp:146-256): per element transpose chains
 * with Hadamard-squared 1D factors, colour-ordered scalar gather, replicate
 * over components, constrained entries 1. */
static void op_diagonal(const Op* op, double* d) {
  const Restr* r = &op->r;
  const Basis* b = op->basis;
  const int nn = b->p + 1, q = b->q, nq = q * q * q, S = r->S;
  const int64_t E = r->E, n_L = r->n_L;
  const int mx = nn > q ? nn : q;
  double* bb = malloc(sizeof(double) * nn * q);
  double* dd = malloc(sizeof(double) * nn * q);
  double* bd = malloc(sizeof(double) * nn * q);
  for (int i = 0; i < nn * q; ++i) {
    bb[i] = b->Bt[i] * b->Bt[i];
    dd[i] = b->Gt[i] * b->Gt[i];
    bd[i] = b->Bt[i] * b->Gt[i];
  }
  double* ediag = calloc((size_t)E * S, sizeof(double));
  double* tmp = malloc(sizeof(double) * S);
  double* ta = malloc(sizeof(double) * mx * mx * mx);
  double* tb = malloc(sizeof(double) * mx * mx * mx);
  for (int64_t e = 0; e < E; ++e) {
    double* diag = ediag + e * S;
    if (op->beta != 0.0) {
      chain3(bb, bb, bb, nn, q, 1, op->mass_qd + e * nq, tmp, ta, tb, 0);
      for (int i = 0; i < S; ++i) diag[i] += op->beta * tmp[i];
    }
    if (op->alpha != 0.0) {
      int s = 0;
      for (int a = 0; a < 3; ++a)
        for (int c = a; c < 3; ++c, ++s) {
          const double* f[3] = {bb, bb, bb};
          for (int k = 0; k < 3; ++k) {
            if (k == a && k == c) f[k] = dd;
            else if (k == a || k == c) f[k] = bd;
          }
          chain3(f[0], f[1], f[2], nn, q, 1, op->diff_qd + (e * 6 + s) * nq, tmp, ta, tb, 0);
          const double w = op->alpha * (a == c ? 1.0 : 2.0);
          for (int i = 0; i < S; ++i) diag[i] += w * tmp[i];
        }
    }
  }
  double* ldiag = malloc(sizeof(double) * n_L);
  apply_gt(r, 1, ediag, ldiag);
  for (int c = 0; c < op->m; ++c) memcpy(d + c * n_L, ldiag, sizeof(double) * n_L);
  for (int c = 0; c < op->m; ++c)
    for (int64_t k = 0; k < op->ncons; ++k) d[c * n_L + op->cons[k]] = 1.0;
  free(bb); free(dd); free(bd); free(ediag); free(tmp); free(ta); free(tb); free(ldiag);
}

/* ------------------------------------------------------------------ PCG
 * dot_deterministic: 4096-element blocks, then a pairwise tree
 * (src/parallel.cpp:69-106). */
static double dot_det(const double* a, const double* b, int64_t n) {
  const int64_t nb = (n + 4095) / 4096;
  if (nb == 0) return 0.0;
  double* part = malloc(sizeof(double) * nb);
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t i0 = k * 4096, i1 = i0 + 4096 < n ? i0 + 4096 : n;
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i) s += a[i] * b[i];
    part[k] = s;
  }
  for (int64_t w = 1; w < nb; w *= 2)
    for (int64_t i = 0; i + w < nb; i += 2 * w) part[i] += part[i + w];
  const double r = part[0];
  free(part);
  return r;
}

/* pcg (src/pcg.cpp:24-115), x0 = 0. */
static int pcg(const Op* op, int64_t n, const double* b, const double* diag, double tol,
               int max_iter, int fixed, double* x, double* hist, int hist_cap, int* iters,
               int* converged) {
  double* r = malloc(sizeof(double) * n);
  double* z = calloc(n, sizeof(double));
  double* p = calloc(n, sizeof(double));
  double* Ap = calloc(n, sizeof(double));
  int nh = 0, conv = 0, rc = 0;
  double last_res = 0.0, target = 0.0;
  memcpy(r, b, sizeof(double) * n);
  for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
#define PUSH(v) do { last_res = (v); if (nh < hist_cap) hist[nh] = last_res; nh++; } while (0)
  const double norm_b = sqrt(dot_det(r, r, n));
  if (!isfinite(norm_b)) { rc = fail(2, "pcg: right-hand side is not finite"); goto done; }
  PUSH(norm_b);
  if (norm_b == 0.0) { conv = 1; goto done; }
  for (int64_t i = 0; i < n; ++i) z[i] = diag ? r[i] / diag[i] : r[i];
  memcpy(p, z, sizeof(double) * n);
  double rho = dot_det(r, z, n);
  const int limit = fixed >= 0 ? fixed : max_iter;
  target = tol * norm_b;
  for (int it = 1; it <= limit; ++it) {
    op_apply(op, p, Ap);
    const double pap = dot_det(p, Ap, n);
    if (!isfinite(pap)) { rc = fail(2, "pcg: NaN in operator apply"); goto done; }
    if (pap <= 0.0) {
      if (rho == 0.0) { conv = 1; break; }
      rc = fail(2, "pcg: indefinite direction (p^T A p <= 0), operator is not SPD");
      goto done;
    }
    const double alpha = rho / pap;
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * Ap[i];
    }
    const double res = sqrt(dot_det(r, r, n));
    if (!isfinite(res)) { rc = fail(2, "pcg: residual is not finite"); goto done; }
    PUSH(res);
    if (res <= target) {
      conv = 1;
      if (fixed < 0) break;
    }
    if (it == limit) break;
    if (res == 0.0) break;
    for (int64_t i = 0; i < n; ++i) z[i] = diag ? r[i] / diag[i] : r[i];
    const double rho_new = dot_det(r, z, n);
    const double beta = rho_new / rho;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_new;
  }
  if (last_res <= target) conv = 1;
done:
#undef PUSH
  *iters = nh > 0 ? nh - 1 : 0;
  *converged = conv;
  free(r); free(z); free(p); free(Ap);
  return rc;
}

/* ------------------------------------------------------------------ BP problem
 * bp_setup (src/bench.cpp:13-119). */
typedef struct {
  int bp, p, m;
  Mesh mesh;
  Basis basis;
  Op op;
  double *mass_qd, *diff_qd;
  double *rhs, *exact;
  int64_t n_dofs;
} Problem;

static double manufactured(double x, double y, double z) {
  return sin(M_PI * x) * sin(M_PI * y) * sin(M_PI * z);
}

void* orc_setup(int bp, int p, int nx, int ny, int nz, int deform, int threads) {
  (void)threads;
  if (bp < 1 || bp > 6) { fail(1, "unknown problem"); return NULL; }
  if (p < 1) { fail(1, "bp_setup: p must be >= 1"); return NULL; }
  if (nx < 1 || ny < 1 || nz < 1) { fail(1, "bp_setup: element counts must be >= 1"); return NULL; }
  Problem* pr = calloc(1, sizeof(Problem));
  pr->bp = bp; pr->p = p;
  pr->m = bp % 2 == 1 ? 1 : 3;
  const int q = bp <= 4 ? p + 2 : p + 1;
  const int kind = bp <= 4 ? 0 : 1;
  const double alpha = bp <= 2 ? 0.0 : 1.0, beta = bp <= 2 ? 1.0 : 0.0;
  mesh_build(&pr->mesh, nx, ny, nz, p, deform);
  basis_make(&pr->basis, p, kind, q);
  if (qdata_compute(&pr->mesh, &pr->basis, 0, &pr->mass_qd)) { orc_free(pr); return NULL; }
  if (alpha > 0 && qdata_compute(&pr->mesh, &pr->basis, 1, &pr->diff_qd)) {
    orc_free(pr);
    return NULL;
  }
  const int64_t n_L = pr->mesh.n_L;
  double* f = malloc(sizeof(double) * pr->m * n_L);
  pr->exact = malloc(sizeof(double) * pr->m * n_L);
  for (int64_t i = 0; i < n_L; ++i) {
    const double x = pr->mesh.coords[i], y = pr->mesh.coords[n_L + i],
                 z = pr->mesh.coords[2 * n_L + i];
    const double u = manufactured(x, y, z);
    const double fv = alpha > 0 ? 3.0 * M_PI * M_PI * manufactured(x, y, z) : u;
    for (int c = 0; c < pr->m; ++c) {
      f[c * n_L + i] = fv;
      pr->exact[c * n_L + i] = u;
    }
  }
  /* b = B f with the unconstrained mass operator (bench.cpp:106-111) */
  Op mass_op = {0};
  restr_make(&mass_op.r, &pr->mesh, pr->m);
  mass_op.basis = &pr->basis;
  mass_op.mass_qd = pr->mass_qd;
  mass_op.m = pr->m;
  mass_op.alpha = 0.0;
  mass_op.beta = 1.0;
  pr->rhs = malloc(sizeof(double) * pr->m * n_L);
  op_apply(&mass_op, f, pr->rhs);
  free(f);
  const int constrained = bp >= 3;
  pr->op = mass_op;
  pr->op.alpha = alpha;
  pr->op.beta = beta;
  pr->op.mass_qd = beta > 0 ? pr->mass_qd : NULL;
  pr->op.diff_qd = pr->diff_qd;
  pr->op.cons = constrained ? pr->mesh.boundary : NULL;
  pr->op.ncons = constrained ? pr->mesh.n_boundary : 0;
  for (int c = 0; c < pr->m; ++c)
    for (int64_t k = 0; k < pr->op.ncons; ++k) pr->rhs[c * n_L + pr->op.cons[k]] = 0.0;
  pr->n_dofs = (int64_t)pr->m * (n_L - pr->op.ncons);
  return pr;
}

void orc_free(void* h) {
  Problem* pr = h;
  if (!pr) return;
  mesh_free(&pr->mesh);
  basis_free(&pr->basis);
  restr_free(&pr->op.r);
  free(pr->mass_qd); free(pr->diff_qd); free(pr->rhs); free(pr->exact);
  free(pr);
}

void orc_info(void* h, int64_t* info) {
  Problem* pr = h;
  info[0] = pr->m;
  info[1] = pr->mesh.n_L;
  info[2] = pr->mesh.E;
  info[3] = pr->op.r.S;
  info[4] = (int64_t)pr->basis.q * pr->basis.q * pr->basis.q;
  info[5] = pr->basis.q;
  info[6] = pr->n_dofs;
  info[7] = pr->op.ncons;
  info[8] = pr->p;
  info[9] = pr->mesh.NX;
}

const double* orc_rhs(void* h) { return ((Problem*)h)->rhs; }
const double* orc_exact(void* h) { return ((Problem*)h)->exact; }
const double* orc_coords(void* h) { return ((Problem*)h)->mesh.coords; }
const int64_t* orc_indices(void* h) { return ((Problem*)h)->op.r.idx; }
const int64_t* orc_constrained(void* h) { return ((Problem*)h)->op.cons; }
const double* orc_qdata(void* h, int kind) {
  Problem* pr = h;
  return kind == 0 ? pr->op.mass_qd : pr->op.diff_qd;
}
const double* orc_interp1d(void* h) { return ((Problem*)h)->basis.B; }
const double* orc_grad1d(void* h) { return ((Problem*)h)->basis.G; }
double orc_alpha(void* h) { return ((Problem*)h)->op.alpha; }
double orc_beta(void* h) { return ((Problem*)h)->op.beta; }

int orc_apply(void* h, const double* x, double* y) {
  op_apply(&((Problem*)h)->op, x, y);
  return 0;
}

int orc_diagonal(void* h, double* d) {
  op_diagonal(&((Problem*)h)->op, d);
  return 0;
}

int orc_solve(void* h, double tol, int max_iter, int jacobi, int fixed_iters, double* x,
              double* hist, int hist_cap, int* iters, int* converged) {
  Problem* pr = h;
  const int64_t n = (int64_t)pr->m * pr->mesh.n_L;
  double* diag = NULL;
  if (jacobi) {
    diag = malloc(sizeof(double) * n);
    op_diagonal(&pr->op, diag);
  }
  const int rc = pcg(&pr->op, n, pr->rhs, diag, tol, max_iter, fixed_iters, x, hist, hist_cap,
                     iters, converged);
  free(diag);
  return rc;
}

/* l2_error (src/bench.cpp:139-189): Gauss q=p+2 rule regardless of the BP. */
int orc_gather_scalar(void* h, const double* e_scalar, int64_t e_len, double* l_scalar,
                      int64_t l_len) {
  const Restr* r = &((Problem*)h)->op.r;
  if (l_len != r->n_L) return fail(1, "gather_scalar: L-vector length mismatch");
  if (e_len != r->E * r->S) return fail(1, "gather_scalar: E-vector length mismatch");
  apply_gt(r, 1, e_scalar, l_scalar);
  return 0;
}

double orc_l2_error(void* h, const double* u) {
  Problem* pr = h;
  const Mesh* mesh = &pr->mesh;
  const int p = mesh->p;
  Basis eb;
  basis_make(&eb, p, 0, p + 2);
  double* qd = NULL;
  qdata_compute(mesh, &eb, 0, &qd);
  Restr r;
  restr_make(&r, mesh, 1);
  const int S = r.S, q = eb.q, nq = q * q * q, mx = p + 2;
  const int64_t n_L = mesh->n_L;
  double* nodal = malloc(sizeof(double) * S);
  double* uq = malloc(sizeof(double) * nq);
  double* xq = malloc(sizeof(double) * 3 * nq);
  double* diff2 = malloc(sizeof(double) * nq);
  double* ta = malloc(sizeof(double) * mx * mx * mx);
  double* tb = malloc(sizeof(double) * mx * mx * mx);
  double err2 = 0.0;
  for (int64_t e = 0; e < r.E; ++e) {
    const int64_t* idx = r.idx + e * S;
    for (int a = 0; a < 3; ++a) {
      for (int s = 0; s < S; ++s) nodal[s] = mesh->coords[a * n_L + idx[s]];
      basis_batch(&eb, 0, 0, 1, nodal, xq + a * nq, ta, tb);
    }
    for (int i = 0; i < nq; ++i) diff2[i] = 0.0;
    for (int c = 0; c < pr->m; ++c) {
      for (int s = 0; s < S; ++s) nodal[s] = u[c * n_L + idx[s]];
      basis_batch(&eb, 0, 0, 1, nodal, uq, ta, tb);
      for (int i = 0; i < nq; ++i) {
        const double d = uq[i] - manufactured(xq[i], xq[nq + i], xq[2 * nq + i]);
        diff2[i] += d * d;
      }
    }
    for (int i = 0; i < nq; ++i) err2 += qd[e * nq + i] * diff2[i];
  }
  free(nodal); free(uq); free(xq); free(diff2); free(ta); free(tb); free(qd);
  restr_free(&r);
  basis_free(&eb);
  return sqrt(err2);
}
