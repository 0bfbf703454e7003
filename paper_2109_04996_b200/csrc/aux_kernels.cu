// API-surface and setup kernels: restriction (K6), batched basis (K7),
// QFunction (K8), geometric factors (compute_qdata) and the Jacobi diagonal.
//
// None of these is on the timed PCG loop.  They therefore follow the
// reference's arithmetic ORDER exactly — contracted index innermost and
// increasing, products and sums rounded separately (__dmul_rn / __dadd_rn:
// no FMA contraction, like the reference's -ffp-contract=off,
// proj/CMakeLists.txt:32-34), colour-ordered G^T accumulation — so their
// results are bitwise equal to the reference's.
#include <cstdio>
#include <cstdlib>

#include "aux_kernels.h"
#include "hxf_device.cuh"

namespace hxf {

namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// One 1-D contraction along `dim` over a whole element block, by all threads
// of the CTA (proj/src/contraction.cpp:14-76 order).  s = input shape.
__device__ void contract_exact(const double* M, int n_out, int n_in, int dim, int s0, int s1,
                               int s2, const double* in, double* out, bool accumulate) {
  const int o0 = dim == 0 ? n_out : s0, o1 = dim == 1 ? n_out : s1, o2 = dim == 2 ? n_out : s2;
  const int total = o0 * o1 * o2;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int a = t % o0, b = (t / o0) % o1, c = t / (o0 * o1);
    double acc = 0.0;
    if (dim == 0) {
      const double* col = in + n_in * (b + s1 * c);
      for (int k = 0; k < n_in; ++k) acc = dadd(acc, dmul(M[a * n_in + k], col[k]));
    } else if (dim == 1) {
      for (int k = 0; k < n_in; ++k) acc = dadd(acc, dmul(M[b * n_in + k], in[a + s0 * (k + s1 * c)]));
    } else {
      for (int k = 0; k < n_in; ++k) acc = dadd(acc, dmul(M[c * n_in + k], in[a + s0 * b + s0 * s1 * k]));
    }
    out[t] = accumulate ? dadd(out[t], acc) : acc;
  }
  __syncthreads();
}

// chain3 (proj/src/contraction.cpp:212-238) for one element.
__device__ void chain3_exact(const double* m0, const double* m1, const double* m2, int nn, int nq,
                             bool transpose, const double* in, double* out, double* ta, double* tb,
                             bool acc_last) {
  if (!transpose) {
    contract_exact(m0, nq, nn, 0, nn, nn, nn, in, ta, false);
    contract_exact(m1, nq, nn, 1, nq, nn, nn, ta, tb, false);
    contract_exact(m2, nq, nn, 2, nq, nq, nn, tb, out, acc_last);
  } else {
    contract_exact(m2, nn, nq, 2, nq, nq, nq, in, ta, false);
    contract_exact(m1, nn, nq, 1, nq, nq, nn, ta, tb, false);
    contract_exact(m0, nn, nq, 0, nq, nn, nn, tb, out, acc_last);
  }
}

struct BasisDev {
  const double *B, *G, *Bt, *Gt;  // q x nn and nn x q
};

// apply_basis_batch (contraction.cpp:248-295), one CTA per element.
__global__ void basis_apply_kernel(BasisDev bs, int nn, int nq, int mode, int dir, int64_t ne,
                                   const double* __restrict__ in, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int mx = nn > nq ? nn : nq;
  double* ta = sm;
  double* tb = sm + mx * mx * mx;
  const int64_t e = blockIdx.x;
  const int64_t nd3 = (int64_t)nn * nn * nn, nq3 = (int64_t)nq * nq * nq;
  if (mode == 0) {
    if (dir == 0)
      chain3_exact(bs.B, bs.B, bs.B, nn, nq, false, in + e * nd3, out + e * nq3, ta, tb, false);
    else
      chain3_exact(bs.Bt, bs.Bt, bs.Bt, nn, nq, true, in + e * nq3, out + e * nd3, ta, tb, false);
    return;
  }
  for (int d = 0; d < 3; ++d) {
    const double* f0 = d == 0 ? (dir ? bs.Gt : bs.G) : (dir ? bs.Bt : bs.B);
    const double* f1 = d == 1 ? (dir ? bs.Gt : bs.G) : (dir ? bs.Bt : bs.B);
    const double* f2 = d == 2 ? (dir ? bs.Gt : bs.G) : (dir ? bs.Bt : bs.B);
    if (dir == 0)
      chain3_exact(f0, f1, f2, nn, nq, false, in + e * nd3, out + (d * ne + e) * nq3, ta, tb, false);
    else
      chain3_exact(f0, f1, f2, nn, nq, true, in + (d * ne + e) * nq3, out + e * nd3, ta, tb, d > 0);
  }
}

// contract_batch (contraction.cpp:177-206 -> contract_sf, :14-76): one output
// entry per thread, grid-stride over the whole batch; contracted index
// innermost and increasing, products and sums rounded separately, so each
// entry is the reference's value bit for bit (accumulate: out += acc).
__global__ void contract_batch_kernel(const double* __restrict__ M, int n_out, int n_in, int dim,
                                      int s0, int s1, int s2, int64_t ne,
                                      const double* __restrict__ in, double* __restrict__ out,
                                      int accumulate) {
  const int o0 = dim == 0 ? n_out : s0, o1 = dim == 1 ? n_out : s1;
  const int o2 = dim == 2 ? n_out : s2;
  const int64_t oe = (int64_t)o0 * o1 * o2, ie = (int64_t)s0 * s1 * s2;
  const int64_t total = ne * oe;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / oe, r = t - e * oe;
    const int a = (int)(r % o0), b = (int)((r / o0) % o1), c = (int)(r / ((int64_t)o0 * o1));
    const double* ein = in + e * ie;
    double acc = 0.0;
    if (dim == 0) {
      const double* col = ein + (int64_t)n_in * (b + (int64_t)s1 * c);
      for (int k = 0; k < n_in; ++k) acc = dadd(acc, dmul(M[(int64_t)a * n_in + k], col[k]));
    } else if (dim == 1) {
      for (int k = 0; k < n_in; ++k)
        acc = dadd(acc, dmul(M[(int64_t)b * n_in + k], ein[a + (int64_t)s0 * (k + (int64_t)s1 * c)]));
    } else {
      const int64_t plane = (int64_t)s0 * s1;
      for (int k = 0; k < n_in; ++k)
        acc = dadd(acc, dmul(M[(int64_t)c * n_in + k], ein[a + (int64_t)s0 * b + plane * k]));
    }
    out[t] = accumulate ? dadd(out[t], acc) : acc;
  }
}

// apply_qf_mass / apply_qf_diffusion (qfunction.cpp:124-162)
__global__ void qf_kernel(int kind, const double* __restrict__ qd, int nq, int64_t e0, int64_t ne,
                          const double* __restrict__ u, double* __restrict__ v) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ne * nq) return;
  if (kind == 0) {
    v[t] = dmul(qd[e0 * nq + t], u[t]);
    return;
  }
  const int64_t e = t / nq, qi = t % nq;
  const double* s = qd + (e0 + e) * 6 * nq + qi;
  const double u0 = u[(0 * ne + e) * nq + qi], u1 = u[(1 * ne + e) * nq + qi],
               u2 = u[(2 * ne + e) * nq + qi];
  const double s00 = s[0], s01 = s[nq], s02 = s[2 * nq], s11 = s[3 * nq], s12 = s[4 * nq],
               s22 = s[5 * nq];
  v[(0 * ne + e) * nq + qi] = dadd(dadd(dmul(s00, u0), dmul(s01, u1)), dmul(s02, u2));
  v[(1 * ne + e) * nq + qi] = dadd(dadd(dmul(s01, u0), dmul(s11, u1)), dmul(s12, u2));
  v[(2 * ne + e) * nq + qi] = dadd(dadd(dmul(s02, u0), dmul(s12, u1)), dmul(s22, u2));
}

__device__ __forceinline__ int64_t elem_node(const Lattice& L, const int* idx, int64_t e, int s) {
  if (idx) return idx[e * L.S + s];
  const int n1 = L.p + 1;
  const int kx = s % n1, ky = (s / n1) % n1, kz = s / (n1 * n1);
  const int64_t ex = e % L.nx, r = e / L.nx, ey = r % L.ny, ez = r / L.ny;
  return (ex * L.p + kx) + L.NX * ((ey * L.p + ky) + L.NY * (ez * L.p + kz));
}

// apply_g (restriction.cpp:28-48): e[(c*E+e)*S+s] = l[c*n_L + idx]
__global__ void restr_gather_kernel(Lattice L, const int* idx, int m, const double* __restrict__ l,
                                    double* __restrict__ ev) {
  const int64_t total = (int64_t)m * L.E * L.S;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t % L.S);
    const int64_t ce = t / L.S, c = ce / L.E, e = ce % L.E;
    ev[t] = l[c * L.n_L + elem_node(L, idx, e, s)];
  }
}

// ---- structured box (no table): one pass, 32-bit fast division --------------
// apply_g on the lattice: entry t = (c, e, s) of the E-vector, written in
// order (coalesced); the l reads of a thread's line are consecutive nodes.
__global__ void restr_gather_box_kernel(Lattice L, int m, const double* __restrict__ l,
                                        double* __restrict__ ev) {
  // (measured: four entries per trip with the loads first is slower, 62 -> 73 us at C3)
  const uint32_t total = (uint32_t)((int64_t)m * L.E * L.S);
  const FastDiv dS((uint32_t)L.S), dE((uint32_t)L.E), dn1((uint32_t)(L.p + 1)),
      dnx((uint32_t)L.nx), dny((uint32_t)L.ny);
  const uint32_t n1 = (uint32_t)(L.p + 1);
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const uint32_t ce = dS.div(t), s = t - ce * (uint32_t)L.S;
    const uint32_t c = dE.div(ce), e = ce - c * (uint32_t)L.E;
    const uint32_t sy = dn1.div(s), kx = s - sy * n1, kz = dn1.div(sy), ky = sy - kz * n1;
    const uint32_t r = dnx.div(e), ex = e - r * (uint32_t)L.nx, ez = dny.div(r), ey = r - ez * (uint32_t)L.ny;
    const int64_t node = (int64_t)(ex * L.p + kx) +
                         L.NX * ((int64_t)(ey * L.p + ky) + L.NY * (int64_t)(ez * L.p + kz));
    ev[t] = __ldg(l + c * L.n_L + node);
  }
}

// The elements (at most two) containing lattice coordinate i along one axis
// of n elements of degree p: element index and local coordinate per parity
// (a node shared by two elements sits in one even and one odd element).
struct AxisOwners {
  int e[2], k[2];  // by parity of the element index; e = -1: none
};
__device__ __forceinline__ AxisOwners axis_owners(int i, int p, int n, const FastDiv& dp) {
  AxisOwners a{{-1, -1}, {0, 0}};
  const int q = (int)dp.div((uint32_t)i), r = i - q * p;
  if (r == 0) {
    if (q - 1 >= 0) { a.e[(q - 1) & 1] = q - 1; a.k[(q - 1) & 1] = p; }
    if (q < n) { a.e[q & 1] = q; a.k[q & 1] = 0; }
  } else {
    a.e[q & 1] = q;
    a.k[q & 1] = r;
  }
  return a;
}

// multiplicity on the lattice: elements per node = product of the per-axis
// counts (the integer the reference's sum of ones gives, exactly)
__global__ void multiplicity_box_kernel(Lattice L, double* __restrict__ mult) {
  const FastDiv dNX((uint32_t)L.NX), dNY((uint32_t)L.NY), dp((uint32_t)L.p);
  for (uint32_t node = blockIdx.x * blockDim.x + threadIdx.x; node < (uint32_t)L.n_L;
       node += gridDim.x * blockDim.x) {
    const uint32_t r = dNX.div(node), ix = node - r * (uint32_t)L.NX, iz = dNY.div(r),
                   iy = r - iz * (uint32_t)L.NY;
    auto cnt = [&](int i, int n) {
      const AxisOwners a = axis_owners(i, L.p, n, dp);
      return (a.e[0] >= 0 ? 1 : 0) + (a.e[1] >= 0 ? 1 : 0);
    };
    mult[node] = (double)(cnt((int)ix, L.nx) * cnt((int)iy, L.ny) * cnt((int)iz, L.nz));
  }
}

// One colour class of apply_g_transpose / gather_scalar (restriction.cpp:50-106):
// elements of one parity class share no node, so plain adds are race-free and
// the per-node accumulation order is the class order.
__global__ void restr_scatter_color_kernel(Lattice L, const int* idx, int m, int color,
                                           int64_t ncol, int64_t cx_n, int64_t cy_n,
                                           const double* __restrict__ ev, double* __restrict__ l) {
  const int64_t total = (int64_t)m * ncol * L.S;
  const int cx = color & 1, cy = (color >> 1) & 1, cz = (color >> 2) & 1;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t % L.S);
    const int64_t ck = t / L.S, c = ck / ncol, k = ck % ncol;
    const int64_t ix = k % cx_n, r = k / cx_n, iy = r % cy_n, iz = r / cy_n;
    const int64_t e = (2 * ix + cx) + L.nx * ((2 * iy + cy) + (int64_t)L.ny * (2 * iz + cz));
    const int64_t node = c * L.n_L + elem_node(L, idx, e, s);
    l[node] = dadd(l[node], ev[(c * L.E + e) * L.S + s]);
  }
}

// G^T for a general (unstructured) table: FP64 RED (order not pinned).
__global__ void restr_scatter_atomic_kernel(Lattice L, const int* idx, int m,
                                            const double* __restrict__ ev, double* __restrict__ l) {
  const int64_t total = (int64_t)m * L.E * L.S;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(t % L.S);
    const int64_t ce = t / L.S, c = ce / L.E, e = ce % L.E;
    red_add(l + c * L.n_L + elem_node(L, idx, e, s), ev[t]);
  }
}

__global__ void multiplicity_kernel(Lattice L, const int* idx, double* __restrict__ mult) {
  const int64_t total = L.E * L.S;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x)
    red_add(mult + elem_node(L, idx, t / L.S, (int)(t % L.S)), 1.0);  // integer sums: exact
}

// compute_qdata, part 1 (qfunction.cpp:37-72): gradients of the three
// coordinate fields for a batch of elements, J[a][d] at (a*3+d)*nb*nq.
__global__ void qdata_grad_kernel(BasisDev bs, Lattice L, const int* idx, int nq1,
                                  const double* __restrict__ coords, int64_t e0, int64_t nb,
                                  double* __restrict__ grad) {
  extern __shared__ double sm[];
  const int nn = L.p + 1, mx = nn > nq1 ? nn : nq1;
  double* ta = sm;
  double* tb = sm + mx * mx * mx;
  double* u = tb + mx * mx * mx;
  const int64_t eb = blockIdx.x, e = e0 + eb;
  const int nq = nq1 * nq1 * nq1;
  for (int a = 0; a < 3; ++a) {
    for (int s = threadIdx.x; s < L.S; s += blockDim.x) u[s] = coords[a * L.n_L + elem_node(L, idx, e, s)];
    __syncthreads();
    for (int d = 0; d < 3; ++d) {
      const double* f0 = d == 0 ? bs.G : bs.B;
      const double* f1 = d == 1 ? bs.G : bs.B;
      const double* f2 = d == 2 ? bs.G : bs.B;
      chain3_exact(f0, f1, f2, nn, nq1, false, u, grad + ((a * 3 + d) * nb + eb) * nq, ta, tb, false);
    }
  }
}

// compute_qdata, part 2 (qfunction.cpp:73-116): det, inverse, w det J^-1 J^-T.
__global__ void qdata_point_kernel(int kind, int nq1, const double* __restrict__ w1,
                                   int64_t e0, int64_t nb, const double* __restrict__ grad,
                                   double* __restrict__ vals, unsigned long long* fail_key,
                                   double* fail_det) {
  const int nq = nq1 * nq1 * nq1;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nb * nq) return;
  const int64_t eb = t / nq;
  const int qi = (int)(t % nq);
  const int64_t e = e0 + eb;
  double J[3][3];
  for (int a = 0; a < 3; ++a)
    for (int d = 0; d < 3; ++d) J[a][d] = grad[((a * 3 + d) * nb + eb) * nq + qi];
  const double det =
      dadd(dsub(dmul(J[0][0], dsub(dmul(J[1][1], J[2][2]), dmul(J[1][2], J[2][1]))),
                dmul(J[0][1], dsub(dmul(J[1][0], J[2][2]), dmul(J[1][2], J[2][0])))),
           dmul(J[0][2], dsub(dmul(J[1][0], J[2][1]), dmul(J[1][1], J[2][0]))));
  if (!(det > 0.0)) {
    const unsigned long long key = (unsigned long long)e * (unsigned long long)nq + qi;
    const unsigned long long old = atomicMin(fail_key, key);
    if (key < old) fail_det[0] = det;  // best effort: message detail only
    return;
  }
  const int qa = qi % nq1, qb = (qi / nq1) % nq1, qc = qi / (nq1 * nq1);
  const double wq = dmul(dmul(w1[qa], w1[qb]), w1[qc]);
  const double wdet = dmul(wq, det);
  if (kind == 0) {
    vals[e * nq + qi] = wdet;
    return;
  }
  double inv[3][3];
  inv[0][0] = __ddiv_rn(dsub(dmul(J[1][1], J[2][2]), dmul(J[1][2], J[2][1])), det);
  inv[0][1] = __ddiv_rn(dsub(dmul(J[0][2], J[2][1]), dmul(J[0][1], J[2][2])), det);
  inv[0][2] = __ddiv_rn(dsub(dmul(J[0][1], J[1][2]), dmul(J[0][2], J[1][1])), det);
  inv[1][0] = __ddiv_rn(dsub(dmul(J[1][2], J[2][0]), dmul(J[1][0], J[2][2])), det);
  inv[1][1] = __ddiv_rn(dsub(dmul(J[0][0], J[2][2]), dmul(J[0][2], J[2][0])), det);
  inv[1][2] = __ddiv_rn(dsub(dmul(J[0][2], J[1][0]), dmul(J[0][0], J[1][2])), det);
  inv[2][0] = __ddiv_rn(dsub(dmul(J[1][0], J[2][1]), dmul(J[1][1], J[2][0])), det);
  inv[2][1] = __ddiv_rn(dsub(dmul(J[0][1], J[2][0]), dmul(J[0][0], J[2][1])), det);
  inv[2][2] = __ddiv_rn(dsub(dmul(J[0][0], J[1][1]), dmul(J[0][1], J[1][0])), det);
  int s = 0;
  for (int a = 0; a < 3; ++a)
    for (int b = a; b < 3; ++b, ++s) {
      const double v = dadd(dadd(dmul(inv[a][0], inv[b][0]), dmul(inv[a][1], inv[b][1])),
                            dmul(inv[a][2], inv[b][2]));
      vals[(e * 6 + s) * nq + qi] = dmul(wdet, v);
    }
}

// Setup fields of the structured box on the device (mesh.cpp:42-78,
// bench.cpp:56-62, 89-105): node coordinates from the 1-D axes and the
// per-axis sines of the undeformed axes (host-computed, glibc), the sine bump
// ((0.05 sx) sy) sz, and the manufactured u* = sin(pi x) sin(pi y) sin(pi z)
// / f = 3 pi^2 u*.  Coordinates are the reference's bit for bit; u*, f too
// on the undeformed box (the axis sines ARE sin(pi x)); on the sine box the
// deformed point's sines come from CUDA's sin (within 1e-15 of max|u| of glibc's).
struct BoxAxes {
  const double *cx, *cy, *cz;  // global 1-D axes (mesh.cpp:12-28)
  const double *sx, *sy, *sz;  // sin(M_PI * c) on those axes
};

__global__ void box_fields_kernel(BoxAxes ax, int64_t NX, int64_t NY, int64_t n_L, int64_t ox,
                                  int64_t oy, int64_t oz, int deform, int m, int poisson,
                                  double* __restrict__ coords, double* __restrict__ f,
                                  double* __restrict__ u) {
  for (int64_t node = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; node < n_L;
       node += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ix = node % NX, r = node / NX, iy = r % NY, iz = r / NY;
    const int64_t gx = ox + ix, gy = oy + iy, gz = oz + iz;
    double x = ax.cx[gx], y = ax.cy[gy], z = ax.cz[gz];
    double uv;
    if (deform) {
      const double bump = dmul(dmul(dmul(0.05, ax.sx[gx]), ax.sy[gy]), ax.sz[gz]);
      x = dadd(x, bump);
      y = dadd(y, bump);
      z = dadd(z, bump);
      uv = dmul(dmul(sin(dmul(M_PI, x)), sin(dmul(M_PI, y))), sin(dmul(M_PI, z)));
    } else {
      uv = dmul(dmul(ax.sx[gx], ax.sy[gy]), ax.sz[gz]);
    }
    if (coords) {
      coords[node] = x;
      coords[n_L + node] = y;
      coords[2 * n_L + node] = z;
    }
    const double fv = poisson ? dmul(dmul(dmul(3.0, M_PI), M_PI), uv) : uv;
    for (int c = 0; c < m; ++c) {
      if (f) f[c * n_L + node] = fv;
      if (u) u[c * n_L + node] = uv;
    }
  }
}

// operator_diagonal element part (operator.cpp:178-244): transpose chains of
// Hadamard-squared 1-D factors over the (unscaled) geometric factors.
struct DiagFactors {
  const double *bb, *dd, *bd;  // nn x q
};

__global__ void diag_elem_kernel(DiagFactors f, int nn, int nq1, const double* __restrict__ mass_qd,
                                 int64_t mass_stride, const double* __restrict__ diff_qd,
                                 int64_t diff_stride, double alpha, double beta,
                                 double* __restrict__ ediag) {
  extern __shared__ double sm[];
  const int mx = nn > nq1 ? nn : nq1;
  double* ta = sm;
  double* tb = sm + mx * mx * mx;
  double* tmp = tb + mx * mx * mx;
  const int S = nn * nn * nn, nq = nq1 * nq1 * nq1;
  const int64_t e = blockIdx.x;
  double* diag = ediag + e * S;
  for (int i = threadIdx.x; i < S; i += blockDim.x) diag[i] = 0.0;
  __syncthreads();
  if (beta != 0.0) {
    chain3_exact(f.bb, f.bb, f.bb, nn, nq1, true, mass_qd + e * mass_stride, tmp, ta, tb, false);
    for (int i = threadIdx.x; i < S; i += blockDim.x) diag[i] = dadd(diag[i], dmul(beta, tmp[i]));
    __syncthreads();
  }
  if (alpha != 0.0) {
    int s = 0;
    for (int a = 0; a < 3; ++a)
      for (int b = a; b < 3; ++b, ++s) {
        const double* g[3] = {f.bb, f.bb, f.bb};
        for (int k = 0; k < 3; ++k) {
          if (k == a && k == b) g[k] = f.dd;
          else if (k == a || k == b) g[k] = f.bd;
        }
        chain3_exact(g[0], g[1], g[2], nn, nq1, true, diff_qd + e * diff_stride + s * nq, tmp, ta,
                     tb, false);
        const double wgt = dmul(alpha, a == b ? 1.0 : 2.0);
        for (int i = threadIdx.x; i < S; i += blockDim.x) diag[i] = dadd(diag[i], dmul(wgt, tmp[i]));
        __syncthreads();
      }
  }
}

__global__ void diag_finish_kernel(int64_t n_L, int m, const double* __restrict__ ldiag,
                                   const uint32_t* cons_mask, double* __restrict__ d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_L;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool cons = cons_mask && ((cons_mask[i >> 5] >> (i & 31)) & 1u);
    const double v = cons ? 1.0 : ldiag[i];
    for (int c = 0; c < m; ++c) d[c * n_L + i] = v;
  }
}

bool box_restriction_disabled() {  // HXF_BOX_RESTRICTION=0: the colour-class kernels (A/B)
  static const bool off = [] {
    const char* v = std::getenv("HXF_BOX_RESTRICTION");
    return v && v[0] == '0';
  }();
  return off;
}

int grid_for(int64_t total, int threads) {
  const int64_t g = (total + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

int chain_smem(int nn, int nq, int extra) {
  const int mx = nn > nq ? nn : nq;
  return (2 * mx * mx * mx + extra) * (int)sizeof(double);
}

cudaError_t set_smem(const void* fn, int bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

}  // namespace

cudaError_t launch_basis_apply(cudaStream_t s, int p, int q, const double* B, const double* G,
                               const double* Bt, const double* Gt, int mode, int dir, int64_t ne,
                               const double* in, double* out) {
  const int nn = p + 1;
  const int smem = chain_smem(nn, q, 0);
  cudaError_t err = set_smem((const void*)basis_apply_kernel, smem);
  if (err != cudaSuccess) return err;
  if (ne == 0) return cudaSuccess;
  basis_apply_kernel<<<(unsigned)ne, 128, smem, s>>>(BasisDev{B, G, Bt, Gt}, nn, q, mode, dir, ne,
                                                     in, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_box_fields(cudaStream_t s, const double* axes, const int64_t gdim[3],
                              const int64_t off[3], const int64_t ldim[3], int deform, int m,
                              int poisson, double* coords, double* f, double* u) {
  BoxAxes ax;
  ax.cx = axes;
  ax.cy = ax.cx + gdim[0];
  ax.cz = ax.cy + gdim[1];
  ax.sx = ax.cz + gdim[2];
  ax.sy = ax.sx + gdim[0];
  ax.sz = ax.sy + gdim[1];
  const int64_t n_L = ldim[0] * ldim[1] * ldim[2];
  box_fields_kernel<<<grid_for(n_L, 256), 256, 0, s>>>(ax, ldim[0], ldim[1], n_L, off[0], off[1],
                                                      off[2], deform, m, poisson, coords, f, u);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_contract_batch(cudaStream_t s, const double* M, int n_out, int n_in, int dim,
                                  const int shape[3], int64_t ne, const double* in, double* out,
                                  bool accumulate) {
  const int64_t oe = (int64_t)shape[0] * shape[1] * shape[2] / n_in * n_out;
  if (ne * oe == 0) return cudaSuccess;
  contract_batch_kernel<<<grid_for(ne * oe, 256), 256, 0, s>>>(M, n_out, n_in, dim, shape[0],
                                                               shape[1], shape[2], ne, in, out,
                                                               accumulate ? 1 : 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_qfunction(cudaStream_t s, int kind, const double* qd, int nq, int64_t e0,
                             int64_t ne, const double* u, double* v) {
  const int64_t total = ne * nq;
  if (total == 0) return cudaSuccess;
  qf_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(kind, qd, nq, e0, ne, u, v);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_restriction(cudaStream_t s, const Lattice& L, const int* idx, bool colorable,
                               int m, bool transpose, const double* in, double* out) {
  // structured box, 32-bit index space: the lattice gather with 32-bit fast
  // division (C3: 95 -> 62 us)
  const bool box32 = !idx && colorable && (int64_t)m * L.E * L.S < (int64_t(1) << 31) &&
                     (int64_t)m * L.n_L < (int64_t(1) << 31) && !box_restriction_disabled();
  // (G^T stays on the colour classes below: a one-pass gather form — each node
  // summing its elements' entries in class order — measured slower, 166 vs 159
  // us at C3)
  if (box32 && !transpose) {
    restr_gather_box_kernel<<<grid_for((int64_t)m * L.E * L.S, 256), 256, 0, s>>>(L, m, in, out);
    count_launch();
    return cudaGetLastError();
  }
  if (!transpose) {
    restr_gather_kernel<<<grid_for((int64_t)m * L.E * L.S, 256), 256, 0, s>>>(L, idx, m, in, out);
    count_launch();
    return cudaGetLastError();
  }
  cudaError_t err = cudaMemsetAsync(out, 0, sizeof(double) * m * L.n_L, s);
  if (err != cudaSuccess) return err;
  if (!colorable) {
    restr_scatter_atomic_kernel<<<grid_for((int64_t)m * L.E * L.S, 256), 256, 0, s>>>(L, idx, m, in,
                                                                                       out);
    count_launch();
    return cudaGetLastError();
  }
  for (int color = 0; color < 8; ++color) {
    const int64_t cx_n = (L.nx - (color & 1) + 1) / 2, cy_n = (L.ny - ((color >> 1) & 1) + 1) / 2,
                  cz_n = (L.nz - ((color >> 2) & 1) + 1) / 2;
    const int64_t ncol = cx_n * cy_n * cz_n;
    if (ncol == 0) continue;
    restr_scatter_color_kernel<<<grid_for((int64_t)m * ncol * L.S, 256), 256, 0, s>>>(
        L, idx, m, color, ncol, cx_n, cy_n, in, out);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t launch_multiplicity(cudaStream_t s, const Lattice& L, const int* idx, double* mult) {
  if (!idx && L.n_L < (int64_t(1) << 31) && !box_restriction_disabled()) {
    multiplicity_box_kernel<<<grid_for(L.n_L, 256), 256, 0, s>>>(L, mult);
    count_launch();
    return cudaGetLastError();
  }
  cudaError_t err = cudaMemsetAsync(mult, 0, sizeof(double) * L.n_L, s);
  if (err != cudaSuccess) return err;
  multiplicity_kernel<<<grid_for(L.E * L.S, 256), 256, 0, s>>>(L, idx, mult);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_qdata(cudaStream_t s, const Lattice& L, const int* idx, int q,
                         const double* B, const double* G, const double* w1,
                         const double* coords, int kind, double* vals, double* scratch,
                         int64_t batch, unsigned long long* fail_key, double* fail_det) {
  const int nn = L.p + 1, nq = q * q * q;
  const int smem = chain_smem(nn, q, nn * nn * nn);
  cudaError_t err = set_smem((const void*)qdata_grad_kernel, smem);
  if (err != cudaSuccess) return err;
  for (int64_t e0 = 0; e0 < L.E; e0 += batch) {
    const int64_t nb = (L.E - e0) < batch ? (L.E - e0) : batch;
    qdata_grad_kernel<<<(unsigned)nb, 128, smem, s>>>(BasisDev{B, G, nullptr, nullptr}, L, idx, q,
                                                      coords, e0, nb, scratch);
    const int64_t npts = nb * nq;
    qdata_point_kernel<<<(unsigned)((npts + 255) / 256), 256, 0, s>>>(kind, q, w1, e0, nb, scratch,
                                                                     vals, fail_key, fail_det);
    count_launch(2);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

cudaError_t launch_diagonal(cudaStream_t s, const Lattice& L, const int* idx, bool colorable, int q,
                            const double* bb, const double* dd, const double* bd,
                            const double* mass_qd, int64_t mass_stride, const double* diff_qd,
                            int64_t diff_stride, double alpha, double beta, int m,
                            const uint32_t* cons_mask, double* ediag, double* ldiag, double* d) {
  const int nn = L.p + 1;
  const int smem = chain_smem(nn, q, nn * nn * nn);
  cudaError_t err = set_smem((const void*)diag_elem_kernel, smem);
  if (err != cudaSuccess) return err;
  diag_elem_kernel<<<(unsigned)L.E, 128, smem, s>>>(DiagFactors{bb, dd, bd}, nn, q, mass_qd,
                                                     mass_stride, diff_qd, diff_stride, alpha, beta,
                                                     ediag);
  count_launch();
  err = launch_restriction(s, L, idx, colorable, 1, true, ediag, ldiag);
  if (err != cudaSuccess) return err;
  diag_finish_kernel<<<grid_for(L.n_L, 256), 256, 0, s>>>(L.n_L, m, ldiag, cons_mask, d);
  count_launch();
  return cudaGetLastError();
}

}  // namespace hxf
