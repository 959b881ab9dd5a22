// geometry.cu -- device-side setup kernels (metric terms, Jacobian interpolant, face checks) and
// small utility kernels (halo pack, deterministic reductions).  Product code.
//
// Metric terms: exact adjugate in 2D, conservative curl form in 3D (column
// reading R4); normals by Nanson's formula J n = G^T nhat; J~ = degree-p_g interpolant of
// det(grad x) at the mapping nodes.  Reference interpolation/derivative matrices come
// from tables.cpp; each CTA handles one element.
#include <cuda_runtime.h>
#include <stdint.h>

#include "geometry.cuh"

namespace esb {

// ---- double-double arithmetic (error-free transformations with FMA) for the setup geometry ----
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  s.lo += a.lo + b.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  double p = a.hi * b.hi;
  double e = fma(a.hi, b.hi, -p);
  e += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p, e);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_sub(dd a, dd b) { return dd_add(a, dd_neg(b)); }

__global__ void geometry_kernel(GeoArgs g) {
  extern __shared__ __align__(16) double sm[];
  const int d = g.dim, Npg = g.Npg, Ncl = g.Ncl, Nq = g.Nq, NF = g.NF, Nqf = g.Nqf;
  const int NG = d * d;
  double* xs = sm;               // [Npg][d] local mapping-node coordinates (exact inputs)
  double* det = xs + Npg * d;    // [Npg][2] dd
  double* rr = det + 2 * Npg;    // [Ncl][9][2] dd
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = tid; k < Npg * d; k += nt) xs[k] = g.xmap[(size_t)e * Npg * d + k];
  __syncthreads();
  // A[m*3+l] = dx_m/dxi_l in double-double
  auto grad_at = [&](const double* Dh, const double* Dl, int npts, int X, dd* A) {
    for (int k = 0; k < 9; ++k) A[k] = {0.0, 0.0};
    for (int l = 0; l < d; ++l) {
      const size_t row = ((size_t)l * npts + X) * Npg;
      for (int i = 0; i < Npg; ++i) {
        dd c = {__ldg(&Dh[row + i]), __ldg(&Dl[row + i])};
        for (int m = 0; m < d; ++m) A[m * 3 + l] = dd_add(A[m * 3 + l], dd_mul(c, dd{xs[i * d + m], 0.0}));
      }
    }
  };
  if (d == 3) {
    for (int c = tid; c < Ncl; c += nt) {  // r1 = x3 grad x2, r2 = x3 grad x1, r3 = x1 grad x2 at lattice
      dd A[9], x[3] = {{0, 0}, {0, 0}, {0, 0}};
      const size_t row = (size_t)c * Npg;
      for (int i = 0; i < Npg; ++i) {
        dd cc = {__ldg(&g.LmapC[row + i]), __ldg(&g.LmapC_lo[row + i])};
        for (int m = 0; m < 3; ++m) x[m] = dd_add(x[m], dd_mul(cc, dd{xs[i * 3 + m], 0.0}));
      }
      grad_at(g.DmapC, g.DmapC_lo, Ncl, c, A);
      for (int l = 0; l < 3; ++l) {
        dd r1 = dd_mul(x[2], A[1 * 3 + l]), r2 = dd_mul(x[2], A[0 * 3 + l]), r3 = dd_mul(x[0], A[1 * 3 + l]);
        rr[(c * 9 + 0 + l) * 2] = r1.hi;
        rr[(c * 9 + 0 + l) * 2 + 1] = r1.lo;
        rr[(c * 9 + 3 + l) * 2] = r2.hi;
        rr[(c * 9 + 3 + l) * 2 + 1] = r2.lo;
        rr[(c * 9 + 6 + l) * 2] = r3.hi;
        rr[(c * 9 + 6 + l) * 2 + 1] = r3.lo;
      }
    }
  }
  for (int i = tid; i < Npg; i += nt) {
    dd A[9];
    grad_at(g.DmapM, g.DmapM_lo, Npg, i, A);
    dd dt;
    if (d == 2) {
      dt = dd_sub(dd_mul(A[0], A[4]), dd_mul(A[1], A[3]));
    } else {
      dd c0 = dd_sub(dd_mul(A[4], A[8]), dd_mul(A[5], A[7]));
      dd c1 = dd_sub(dd_mul(A[3], A[8]), dd_mul(A[5], A[6]));
      dd c2 = dd_sub(dd_mul(A[3], A[7]), dd_mul(A[4], A[6]));
      dt = dd_add(dd_sub(dd_mul(A[0], c0), dd_mul(A[1], c1)), dd_mul(A[2], c2));
    }
    det[2 * i] = dt.hi;
    det[2 * i + 1] = dt.lo;
    if (!(dt.hi > 0.0)) atomicOr(g.bad, 1);
  }
  __syncthreads();
  auto metric = [&](const double* Dh2, const double* Dl2, const double* Ch, const double* Cl, int npts, int X,
                    double* G) {
    if (d == 2) {
      dd A[9];
      grad_at(Dh2, Dl2, npts, X, A);
      G[0] = A[4].hi;   // G_11 = dx2/dxi2   (P:335 adjugate)
      G[1] = -A[1].hi;  // G_12 = -dx1/dxi2
      G[2] = -A[3].hi;  // G_21 = -dx2/dxi1
      G[3] = A[0].hi;   // G_22 = dx1/dxi1
    } else {
      dd dr[27];  // dr[f*3+l] = d r_f / d xi_l
      for (int k = 0; k < 27; ++k) dr[k] = {0.0, 0.0};
      for (int l = 0; l < 3; ++l) {
        const size_t row = ((size_t)l * npts + X) * Ncl;
        for (int c = 0; c < Ncl; ++c) {
          dd cc = {__ldg(&Ch[row + c]), __ldg(&Cl[row + c])};
          for (int f = 0; f < 9; ++f)
            dr[f * 3 + l] = dd_add(dr[f * 3 + l], dd_mul(cc, dd{rr[(c * 9 + f) * 2], rr[(c * 9 + f) * 2 + 1]}));
        }
      }
      for (int rk = 0; rk < 3; ++rk) {  // columns: -curl r1, curl r2, curl r3 (R4)
        const dd* q = dr + rk * 9;       // q[comp*3 + l]
        dd c0 = dd_sub(q[2 * 3 + 1], q[1 * 3 + 2]);
        dd c1 = dd_sub(q[0 * 3 + 2], q[2 * 3 + 0]);
        dd c2 = dd_sub(q[1 * 3 + 0], q[0 * 3 + 1]);
        double s = rk == 0 ? -1.0 : 1.0;
        G[0 * 3 + rk] = s * c0.hi;
        G[1 * 3 + rk] = s * c1.hi;
        G[2 * 3 + rk] = s * c2.hi;
      }
    }
  };
  for (int X = tid; X < Nq; X += nt) {
    double G[9];
    metric(g.DmapV, g.DmapV_lo, g.DcurlV, g.DcurlV_lo, Nq, X, G);
    dd jt = {0.0, 0.0}, x[3] = {{0, 0}, {0, 0}, {0, 0}};
    const size_t row = (size_t)X * Npg;
    for (int i = 0; i < Npg; ++i) {
      dd c = {__ldg(&g.LmapV[row + i]), __ldg(&g.LmapV_lo[row + i])};
      jt = dd_add(jt, dd_mul(c, dd{det[2 * i], det[2 * i + 1]}));
      for (int m = 0; m < d; ++m) x[m] = dd_add(x[m], dd_mul(c, dd{xs[i * d + m], 0.0}));
    }
    if (!(jt.hi > 0.0)) atomicOr(g.bad, 2);
    double* gv = g.geo_vol + (size_t)e * g.gv_stride;
    for (int k = 0; k < NG; ++k) gv[k * Nq + X] = G[k];
    double W = __ldg(&g.Wvol[X]);
    gv[NG * Nq + X] = W * jt.hi;
    gv[(NG + 1) * Nq + X] = W / jt.hi;
    for (int m = 0; m < d; ++m) g.xq[((size_t)e * Nq + X) * d + m] = x[m].hi + g.shift[(size_t)e * d + m];
    if (g.jt_out) g.jt_out[(size_t)e * Nq + X] = jt.hi;
  }
  for (int F = tid; F < NF; F += nt) {
    double G[9];
    metric(g.DmapF, g.DmapF_lo, g.DcurlF, g.DcurlF_lo, NF, F, G);
    int z = F / Nqf, f = F % Nqf;
    for (int m = 0; m < d; ++m) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += G[l * d + m] * __ldg(&g.nhat[z * 3 + l]);
      g.geo_face[(((size_t)e * (d + 1) + z) * d + m) * Nqf + f] = s;
    }
  }
}

// B J n must be equal and opposite at matched facet nodes (P:736-741 [eq:weights_match])
__global__ void face_check_kernel(FaceCheckArgs a) {
  int64_t e = blockIdx.x;
  const int d = a.dim, n = a.n, Nqf = a.Nqf, Nf = d + 1;
  for (int F = threadIdx.x; F < Nf * Nqf; F += blockDim.x) {
    int z = F / Nqf, f = F % Nqf;
    int64_t slot = a.face_slot[e * Nf + z];
    if (slot >= a.nloc * Nf) continue;  // remote neighbour: checked by its owner
    int64_t o = slot / Nf;
    int zo = (int)(slot % Nf);
    int rf = a.face_reflect[e * Nf + z];
    int fo = d == 2 ? (rf ? n - 1 - f : f) : (rf ? (n - 1 - f % n) + n * (f / n) : f);
    double s2 = 0.0, na = 0.0;
    for (int m = 0; m < d; ++m) {
      double x = a.Bf[z * Nqf + f] * a.geo_face[((e * Nf + z) * d + m) * Nqf + f];
      double y = a.Bf[zo * Nqf + fo] * a.geo_face[((o * Nf + zo) * d + m) * Nqf + fo];
      s2 += (x + y) * (x + y);
      na += x * x;
    }
    double rel = sqrt(s2 / na);
    unsigned long long bits = (unsigned long long)__double_as_longlong(rel);
    atomicMax(a.max_mismatch, bits);
  }
}

// gather local face traces for the halo send buffer
__global__ void pack_kernel(const double* trace, const int64_t* slots, int64_t nsend, int per_face, double* buf) {
  int64_t total = nsend * per_face;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total; k += (int64_t)gridDim.x * blockDim.x) {
    int64_t h = k / per_face;
    buf[k] = trace[slots[h] * per_face + k % per_face];
  }
}

// deterministic fixed-order reduction of per-element partials part[ne][w] -> out[w]
__global__ void reduce_parts_kernel(const double* part, int64_t ne, int w, double* out) {
  __shared__ double red[256];
  for (int c = 0; c < w; ++c) {
    double s = 0.0;
    for (int64_t e = threadIdx.x; e < ne; e += blockDim.x) s += part[e * w + c];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[c] = red[0];
    __syncthreads();
  }
}

// Runge-Kutta stage input / solution: out = y0 + sum_j c_j k_j (k and c by value)
__global__ void rk_comb_kernel(const double* __restrict__ y0, RkComb kc, double* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < kc.nk; ++j) s = fma(kc.c[j], kc.k[j][i], s);
    out[i] = y0[i] + s;
  }
}
// scaled squared error partials (Hairer-Norsett-Wanner I, eq. II.4.11), block-fixed order
__global__ void __launch_bounds__(256) rk_err_kernel(const double* __restrict__ y0, const double* __restrict__ y1,
                                                     RkComb ec, double rtol, double atol, int64_t n, double* part) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double e = 0.0;
    for (int j = 0; j < ec.nk; ++j) e = fma(ec.c[j], ec.k[j][i], e);
    const double sc = atol + rtol * fmax(fabs(y0[i]), fabs(y1[i]));
    const double r = e == 0.0 ? 0.0 : e / sc;  // atol = 0 with a coefficient that stays 0: no 0/0
    s = fma(r, r, s);
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

cudaError_t launch_rk_comb(const double* y0, const RkComb& kc, double* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t b = (n + 255) / 256;
  rk_comb_kernel<<<(unsigned)(b < 148 * 16 ? b : 148 * 16), 256, 0, st>>>(y0, kc, out, n);
  return cudaGetLastError();
}
cudaError_t launch_rk_err(const double* y0, const double* y1, const RkComb& ec, double rtol, double atol,
                          int64_t n, double* part, cudaStream_t st) {
  rk_err_kernel<<<RK_ERR_BLOCKS, 256, 0, st>>>(y0, y1, ec, rtol, atol, n, part);
  return cudaGetLastError();
}

cudaError_t launch_geometry(const GeoArgs& g, int64_t ne, cudaStream_t st) {
  if (ne <= 0) return cudaSuccess;
  size_t sm = ((size_t)g.Npg * g.dim + 2 * (size_t)g.Npg + (size_t)g.Ncl * 18) * sizeof(double);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(geometry_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
  }
  geometry_kernel<<<(unsigned)ne, 128, sm, st>>>(g);
  return cudaGetLastError();
}
__global__ void __launch_bounds__(256) metric_modal_kernel(MetricModalArgs a) {
  const int NG = a.dim * a.dim, n = a.n;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.ne * NG * a.Np) return;
  const int64_t e = t / (NG * a.Np);
  const int r = (int)(t - e * NG * a.Np), lm = r / a.Np, k = r - lm * a.Np;
  const int pr = a.mode_pr[k], a1 = a.pair_a1[pr];
  const int a2 = a.dim == 2 ? k - a.pair_off[pr] : a.pair_a2[pr];
  const int a3 = a.dim == 3 ? k - a.pair_off[pr] : 0, s = a1 + a2;
  const double* G = a.geo_vol + (size_t)e * a.gv_stride + (size_t)lm * a.Nq;
  const int nc = a.dim == 3 ? n : 1;
  double acc = 0.0;
  for (int c = 0; c < nc; ++c) {
    const double p3 = a.dim == 3 ? a.psi3[(s * n + a3) * n + c] : 1.0;
    for (int b = 0; b < n; ++b) {
      const double p23 = a.psi2[(a1 * n + a2) * n + b] * p3;
      for (int q = 0; q < n; ++q) {
        const int i = q + n * b + n * n * c;  // volume node order: eta1 fastest (R9)
        acc = fma(a.psi1[a1 * n + q] * p23 * a.Wvol[i], G[i], acc);
      }
    }
  }
  a.gmod[(size_t)e * a.gm_stride + (size_t)lm * a.Np + k] = acc;
}
cudaError_t launch_metric_modal(const MetricModalArgs& a, cudaStream_t st) {
  const int64_t n = a.ne * a.dim * a.dim * a.Np;
  if (n <= 0) return cudaSuccess;
  metric_modal_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_face_check(const FaceCheckArgs& a, cudaStream_t st) {
  if (a.nloc <= 0) return cudaSuccess;
  face_check_kernel<<<(unsigned)a.nloc, 128, 0, st>>>(a);
  return cudaGetLastError();
}
cudaError_t launch_pack(const double* trace, const int64_t* slots, int64_t nsend, int per_face, double* buf,
                        cudaStream_t st) {
  if (nsend <= 0) return cudaSuccess;
  int64_t total = nsend * per_face;
  unsigned blocks = (unsigned)((total + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  pack_kernel<<<blocks, 256, 0, st>>>(trace, slots, nsend, per_face, buf);
  return cudaGetLastError();
}
cudaError_t launch_reduce_parts(const double* part, int64_t ne, int w, double* out, cudaStream_t st) {
  reduce_parts_kernel<<<1, 256, 0, st>>>(part, ne, w, out);
  return cudaGetLastError();
}

// one thread per (element, point); the element's modal coefficients staged in shared memory
__global__ void __launch_bounds__(128) eval_points_kernel(EvalPtsArgs a) {
  extern __shared__ double su[];
  const int64_t e = blockIdx.y;
  const int nm = a.NC * a.Np;
  for (int k = threadIdx.x; k < nm; k += blockDim.x) su[k] = a.um[e * nm + k];
  __syncthreads();
  const int pt = blockIdx.x * blockDim.x + threadIdx.x;
  if (pt >= a.npts) return;
  const double* pk = a.pkd + (size_t)pt * a.Np;
  for (int v = 0; v < a.NC; ++v) {
    double s = 0.0;
    for (int k = 0; k < a.Np; ++k) s = fma(su[v * a.Np + k], __ldg(pk + k), s);
    a.u[((size_t)e * a.npts + pt) * a.NC + v] = s;
  }
  const double* X = a.xmap + (size_t)e * a.Npg * a.dim;
  if (a.x) {
    for (int m = 0; m < a.dim; ++m) {
      double s = 0.0;
      for (int i = 0; i < a.Npg; ++i) s = fma(__ldg(a.lmap + (size_t)pt * a.Npg + i), X[i * a.dim + m], s);
      a.x[((size_t)e * a.npts + pt) * a.dim + m] = s;
    }
  }
  if (a.jac) {
    double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};  // A[m][l] = d x_m / d xi_l
    for (int l = 0; l < a.dim; ++l)
      for (int i = 0; i < a.Npg; ++i) {
        const double g = __ldg(a.dmap + ((size_t)l * a.npts + pt) * a.Npg + i);
        for (int m = 0; m < a.dim; ++m) A[m][l] = fma(g, X[i * a.dim + m], A[m][l]);
      }
    const double J = a.dim == 2 ? A[0][0] * A[1][1] - A[0][1] * A[1][0]
                                : A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) -
                                      A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                                      A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
    a.jac[(size_t)e * a.npts + pt] = J;
  }
}

cudaError_t launch_eval_points(const EvalPtsArgs& a, cudaStream_t st) {
  if (a.ne <= 0 || a.npts <= 0) return cudaSuccess;
  const size_t sm = (size_t)a.NC * a.Np * sizeof(double);
  dim3 grid((unsigned)((a.npts + 127) / 128), (unsigned)a.ne);
  eval_points_kernel<<<grid, 128, sm, st>>>(a);
  return cudaGetLastError();
}

}  // namespace esb
