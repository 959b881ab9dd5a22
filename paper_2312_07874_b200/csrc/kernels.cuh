// kernels.cuh -- sm_100a kernels of the ES modal DSEM right-hand side (product code).
//
// K1 project_kernel   : u~ -> u = V u~ -> W(u) -> w~ = V^T W/J~ V V^T W J~ W(u) -> w = V w~,
//                       w_f = R w -> entropy-projected states U(w), U(w_f)
// K2 rhs_kernel       : line-wise volume flux differencing, facet correction
//                       (P:525), interface flux, lifting and the
//                       weight-adjusted inverse mass matrix, fused RK4 stage epilogue.
// One CTA per element; all per-element work is staged in shared memory; FP64 throughout.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace esb {

// ------------------------------------------------------------------------------------------------
// compile-time sizes
// ------------------------------------------------------------------------------------------------
template <int DIM, int N>
struct Sz {
  static constexpr int P = N - 1;
  static constexpr int Nq = DIM == 2 ? N * N : N * N * N;
  static constexpr int Nf = DIM + 1;
  static constexpr int Nqf = DIM == 2 ? N : N * N;
  static constexpr int NF = Nf * Nqf;
  static constexpr int Np = DIM == 2 ? N * (N + 1) / 2 : N * (N + 1) * (N + 2) / 6;
  static constexpr int NPAIR = DIM == 2 ? N : N * (N + 1) / 2;
  static constexpr int NC = DIM + 2;
  static constexpr int NG = DIM * DIM;
  static constexpr int NGV = NG + 2;  // G_lm, W J~, W / J~
  static constexpr int GVS = (NGV * Nq + 1) & ~1;  // geo_vol element stride (even, 16-B aligned)
  static constexpr int PRS = (NC * Nq + 1) & ~1;   // prim element stride
  static constexpr int KPT = (Nq + 383) / 384;
  static constexpr int NT = ((Nq + KPT - 1) / KPT + 31) / 32 * 32;
};

// device copy of the reference tables (pointers into one device allocation)
struct DevRef {
  const double *eta, *w, *eta3, *w3;
  const double *skQ1, *skA1, *skA2, *skA3, *skA4;
  const double *lL, *lR, *l3L, *lint4;
  const double *psi1, *psi2, *psi3;
  const int *pair_a1, *pair_a2, *pair_off, *mode_pr, *mode_last;
  const double *Bf, *nhat, *Wvol;
};

struct ProjArgs {
  int64_t n_elem;
  const int64_t* elem_list;  // optional element subset
  const double* u;           // [nloc][NC][Np] modal stage input
  const double* geo_vol;     // [nloc][GVS]: [NGV][Nq] + pad
  double* prim;              // [nloc][PRS]: [NC][Nq] + pad, entropy-projected primitive (rho, v, p)
  double* trace;             // [slots][NC][Nqf] entropy-projected primitive at facet nodes
  double* wt;                // optional [nloc][NC][Np] projected entropy variables w~
  int* bad;                  // admissibility flag
  double gamma;
};

struct RhsArgs {
  int64_t n_elem;
  const int64_t* elem_list;
  const double* prim;
  const double* trace;
  const double* geo_vol;
  const double* geo_face;     // [nloc][Nf][DIM][Nqf] J n = G^T nhat
  const int64_t* face_slot;   // [nloc][Nf]
  const int* face_reflect;    // [nloc][Nf]
  double gamma;
  int es;                     // 1: add local Lax-Friedrichs dissipation
  int mode;                   // 0 dudt, 1..4 RK stage 0..3, 5 dudt + entropy partials
  double* out;                // dudt [nloc][NC][Np]
  const double* u0;           // RK state
  double* acc;                // RK accumulator
  double* ustage;             // RK stage input (written)
  double dt;
  const double* wt;           // entropy mode: w~
  double* part;               // entropy mode: [nloc][2 + NC]
  double c0;                  // value of the constant PKD mode (1/sqrt|ref|)
};

// ------------------------------------------------------------------------------------------------
// physics (reading R3 for the energy component, R5 for the log mean)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ double ln_mean(double x, double y) {
  double f2 = (x * (x - 2.0 * y) + y * y) / (x * (x + 2.0 * y) + y * y);
  if (f2 < 1e-4) return (x + y) / (2.0 + f2 * (2.0 / 3.0 + f2 * (2.0 / 5.0 + f2 * (2.0 / 7.0))));
  return (y - x) / log(y / x);
}
__device__ __forceinline__ double inv_ln_mean(double x, double y) {
  double f2 = (x * (x - 2.0 * y) + y * y) / (x * (x + 2.0 * y) + y * y);
  if (f2 < 1e-4) return (2.0 + f2 * (2.0 / 3.0 + f2 * (2.0 / 5.0 + f2 * (2.0 / 7.0)))) / (x + y);
  return log(y / x) / (y - x);
}

// Ranocha EC flux in direction n: F = sum_m n_m f#_m(a, b)   (P:834 + R3)
template <int DIM>
__device__ __forceinline__ void ec_flux(double ra, const double* va, double pa, double ba, double rb,
                                        const double* vb, double pb, double bb, const double* n,
                                        double gm1inv, double* F) {
  double rho_ln = ln_mean(ra, rb);
  double ib_ln = inv_ln_mean(ba, bb);
  double vn = 0.0, van = 0.0, vbn = 0.0, vdot = 0.0, vav[DIM];
#pragma unroll
  for (int m = 0; m < DIM; ++m) {
    vav[m] = 0.5 * (va[m] + vb[m]);
    vn += vav[m] * n[m];
    van += va[m] * n[m];
    vbn += vb[m] * n[m];
    vdot += va[m] * vb[m];
  }
  double pav = 0.5 * (pa + pb);
  double fr = rho_ln * vn;
  F[0] = fr;
#pragma unroll
  for (int m = 0; m < DIM; ++m) F[1 + m] = fr * vav[m] + pav * n[m];
  F[DIM + 1] = fr * (0.5 * vdot + ib_ln * gm1inv) + 0.5 * (pa * vbn + pb * van);
}

// conservative variables from primitive (for the Lax-Friedrichs jump)
template <int DIM>
__device__ __forceinline__ void cons_of(double r, const double* v, double p, double gm1inv, double* U) {
  double ke = 0.0;
  U[0] = r;
#pragma unroll
  for (int m = 0; m < DIM; ++m) {
    U[1 + m] = r * v[m];
    ke += v[m] * v[m];
  }
  U[DIM + 1] = p * gm1inv + 0.5 * r * ke;
}

// ------------------------------------------------------------------------------------------------
// sum-factorised PKD transforms, NV variables at once, block-wide.
// The principal-function tables are staged in shared memory (PsiS); every work item produces one
// output fiber (all N entries along the output index) from N inputs held in registers, with fully
// unrolled compile-time loops; entries outside the triangular/tetrahedral index range are zero in
// the tables and the matching inputs are predicated to zero.
// ------------------------------------------------------------------------------------------------
struct PsiS {
  const double* p1;  // [a1][a]
  const double* p2;  // [a1][a2][b]
  const double* p3;  // [s][a3][c]   (tet)
  const int* pa1;    // pair -> a1   (tet: (a1,a2) pairs in a1-major order; tri: pair = a1)
  const int* pa2;    // pair -> a2
  const int* poff;   // pair -> first modal index
};

template <int DIM, int N>
__host__ __device__ constexpr int psi_smem_doubles() {
  return N * N + N * N * N + (DIM == 3 ? N * N * N : 0) + (3 * (DIM == 2 ? N : N * (N + 1) / 2) + 1) / 2 + 1;
}

// stage the tables of R into shared memory at `buf` (psi_smem_doubles<DIM,N>() doubles)
template <int DIM, int N>
__device__ PsiS stage_psi(const DevRef& R, double* buf) {
  constexpr int NPAIR = DIM == 2 ? N : N * (N + 1) / 2;
  double* p1 = buf;
  double* p2 = p1 + N * N;
  double* p3 = p2 + N * N * N;
  int* pi = (int*)(p3 + (DIM == 3 ? N * N * N : 0));
  for (int k = threadIdx.x; k < N * N; k += blockDim.x) p1[k] = R.psi1[k];
  for (int k = threadIdx.x; k < N * N * N; k += blockDim.x) {
    p2[k] = R.psi2[k];
    if constexpr (DIM == 3) p3[k] = R.psi3[k];
  }
  for (int k = threadIdx.x; k < NPAIR; k += blockDim.x) {
    pi[k] = R.pair_a1[k];
    pi[NPAIR + k] = R.pair_a2[k];
    pi[2 * NPAIR + k] = R.pair_off[k];
  }
  return PsiS{p1, p2, p3, pi, pi + NPAIR, pi + 2 * NPAIR};
}

template <int DIM, int N, int NV>
__device__ void modal_to_nodal(const PsiS& T, const double* um, double* un, double* t1, double* t2) {
  using S = Sz<DIM, N>;
  constexpr int P = N - 1, NPAIR = S::NPAIR, Np = S::Np, Nq = S::Nq;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (DIM == 2) {
    for (int it = tid; it < N * NV; it += nt) {  // t1[v][a1][b] = sum_a2 psi2[a1][a2][b] u[v][off(a1)+a2]
      const int a1 = it / NV, v = it - a1 * NV;
      const double* src = um + v * Np + T.poff[a1];
      double x[N];
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) x[a2] = (a2 <= P - a1) ? src[a2] : 0.0;
      const double* ps = T.p2 + a1 * N * N;
      double* dst = t1 + (v * N + a1) * N;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) acc = fma(ps[a2 * N + b], x[a2], acc);
        dst[b] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < NV * N; it += nt) {  // u[v][a + N b] = sum_a1 psi1[a1][a] t1[v][a1][b]
      const int v = it / N, b = it - v * N;
      double x[N];
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) x[a1] = t1[(v * N + a1) * N + b];
      double* dst = un + v * Nq + N * b;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int a1 = 0; a1 < N; ++a1) acc = fma(T.p1[a1 * N + a], x[a1], acc);
        dst[a] = acc;
      }
    }
    __syncthreads();
  } else {
    for (int it = tid; it < NPAIR * NV; it += nt) {  // t1[v][pr][c] = sum_a3 psi3[s][a3][c] u[v][off+a3]
      const int pr = it / NV, v = it - pr * NV;
      const int sdeg = T.pa1[pr] + T.pa2[pr];
      const double* src = um + v * Np + T.poff[pr];
      double x[N];
#pragma unroll
      for (int a3 = 0; a3 < N; ++a3) x[a3] = (a3 <= P - sdeg) ? src[a3] : 0.0;
      const double* ps = T.p3 + sdeg * N * N;
      double* dst = t1 + (v * NPAIR + pr) * N;
#pragma unroll
      for (int c = 0; c < N; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int a3 = 0; a3 < N; ++a3) acc = fma(ps[a3 * N + c], x[a3], acc);
        dst[c] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < N * NV * N; it += nt) {  // t2[v][a1][c][b] = sum_a2 psi2[a1][a2][b] t1[v][pr(a1,a2)][c]
      const int a1 = it / (NV * N), r = it - a1 * NV * N, v = r / N, c = r - v * N;
      const int prs = a1 * N - a1 * (a1 - 1) / 2;
      const double* src = t1 + (v * NPAIR + prs) * N + c;
      double x[N];
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) x[a2] = (a2 <= P - a1) ? src[a2 * N] : 0.0;
      const double* ps = T.p2 + a1 * N * N;
      double* dst = t2 + ((v * N + a1) * N + c) * N;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double acc = 0.0;
#pragma unroll
        for (int a2 = 0; a2 < N; ++a2) acc = fma(ps[a2 * N + b], x[a2], acc);
        dst[b] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < NV * N * N; it += nt) {  // u[v][a + N bc] = sum_a1 psi1[a1][a] t2[v][a1][bc]
      const int v = it / (N * N), bc = it - v * N * N;
      double x[N];
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) x[a1] = t2[(v * N + a1) * N * N + bc];
      double* dst = un + v * Nq + N * bc;
#pragma unroll
      for (int a = 0; a < N; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int a1 = 0; a1 < N; ++a1) acc = fma(T.p1[a1 * N + a], x[a1], acc);
        dst[a] = acc;
      }
    }
    __syncthreads();
  }
}

template <int DIM, int N, int NV>
__device__ void nodal_to_modal(const PsiS& T, const double* y, double* um, double* t1, double* t2) {
  using S = Sz<DIM, N>;
  constexpr int P = N - 1, NPAIR = S::NPAIR, Np = S::Np, Nq = S::Nq;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (DIM == 2) {
    for (int it = tid; it < NV * N; it += nt) {  // s1[v][a1][b] = sum_a psi1[a1][a] y[v][a + N b]
      const int v = it / N, b = it - v * N;
      double x[N];
      const double* src = y + v * Nq + N * b;
#pragma unroll
      for (int a = 0; a < N; ++a) x[a] = src[a];
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) acc = fma(T.p1[a1 * N + a], x[a], acc);
        t1[(v * N + a1) * N + b] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < N * NV; it += nt) {  // u[v][off(a1)+a2] = sum_b psi2[a1][a2][b] s1[v][a1][b]
      const int a1 = it / NV, v = it - a1 * NV;
      double x[N];
      const double* src = t1 + (v * N + a1) * N;
#pragma unroll
      for (int b = 0; b < N; ++b) x[b] = src[b];
      const double* ps = T.p2 + a1 * N * N;
      double* dst = um + v * Np + T.poff[a1];
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) {
        if (a2 > P - a1) break;
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) acc = fma(ps[a2 * N + b], x[b], acc);
        dst[a2] = acc;
      }
    }
    __syncthreads();
  } else {
    for (int it = tid; it < NV * N * N; it += nt) {  // s2[v][a1][bc] = sum_a psi1[a1][a] y[v][a + N bc]
      const int v = it / (N * N), bc = it - v * N * N;
      double x[N];
      const double* src = y + v * Nq + N * bc;
#pragma unroll
      for (int a = 0; a < N; ++a) x[a] = src[a];
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) {
        double acc = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) acc = fma(T.p1[a1 * N + a], x[a], acc);
        t2[(v * N + a1) * N * N + bc] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < N * NV * N; it += nt) {  // s1[v][pr(a1,a2)][c] = sum_b psi2[a1][a2][b] s2[v][a1][c][b]
      const int a1 = it / (NV * N), r = it - a1 * NV * N, v = r / N, c = r - v * N;
      const int prs = a1 * N - a1 * (a1 - 1) / 2;
      double x[N];
      const double* src = t2 + ((v * N + a1) * N + c) * N;
#pragma unroll
      for (int b = 0; b < N; ++b) x[b] = src[b];
      const double* ps = T.p2 + a1 * N * N;
      double* dst = t1 + (v * NPAIR + prs) * N + c;
#pragma unroll
      for (int a2 = 0; a2 < N; ++a2) {
        if (a2 > P - a1) break;
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) acc = fma(ps[a2 * N + b], x[b], acc);
        dst[a2 * N] = acc;
      }
    }
    __syncthreads();
    for (int it = tid; it < NPAIR * NV; it += nt) {  // u[v][off+a3] = sum_c psi3[s][a3][c] s1[v][pr][c]
      const int pr = it / NV, v = it - pr * NV;
      const int sdeg = T.pa1[pr] + T.pa2[pr];
      double x[N];
      const double* src = t1 + (v * NPAIR + pr) * N;
#pragma unroll
      for (int c = 0; c < N; ++c) x[c] = src[c];
      const double* ps = T.p3 + sdeg * N * N;
      double* dst = um + v * Np + T.poff[pr];
#pragma unroll
      for (int a3 = 0; a3 < N; ++a3) {
        if (a3 > P - sdeg) break;
        double acc = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) acc = fma(ps[a3 * N + c], x[c], acc);
        dst[a3] = acc;
      }
    }
    __syncthreads();
  }
}

template <int DIM, int N>
__host__ __device__ constexpr int t1_size() {
  using S = Sz<DIM, N>;
  return DIM == 2 ? S::NC * N * N : S::NC * S::NPAIR * N;
}
template <int DIM, int N>
__host__ __device__ constexpr int t2_size() {
  using S = Sz<DIM, N>;
  return DIM == 2 ? 0 : S::NC * S::Nq;
}

// ------------------------------------------------------------------------------------------------
// K1: entropy projection and traces
// ------------------------------------------------------------------------------------------------
template <int DIM, int N>
__host__ __device__ constexpr size_t project_smem_doubles() {
  using S = Sz<DIM, N>;
  return (size_t)S::NC * S::Np + (size_t)S::NC * S::Nq + t1_size<DIM, N>() + t2_size<DIM, N>() +
         (size_t)S::NC * S::NF + psi_smem_doubles<DIM, N>();
}

template <int DIM, int N>
__global__ void __launch_bounds__(Sz<DIM, N>::NT) project_kernel(DevRef R, ProjArgs A) {
  using S = Sz<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf;
  extern __shared__ double sm[];
  double* um = sm;
  double* X = um + NC * Np;
  double* T1 = X + NC * Nq;
  double* T2 = T1 + t1_size<DIM, N>();
  double* FW = T2 + t2_size<DIM, N>();
  const PsiS T = stage_psi<DIM, N>(R, FW + NC * NF);
  const int64_t e = A.elem_list ? A.elem_list[blockIdx.x] : (int64_t)blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double g = A.gamma, gm1 = g - 1.0, gm1inv = 1.0 / gm1;
  const double* gv = A.geo_vol + (size_t)e * S::GVS;
  for (int k = tid; k < NC * Np; k += nt) um[k] = A.u[(size_t)e * NC * Np + k];
  __syncthreads();
  modal_to_nodal<DIM, N, NC>(T, um, X, T1, T2);  // u = V u~
  int bad = 0;
  for (int i = tid; i < Nq; i += nt) {  // W J~ W(u)   (App. B formulas, R7)
    double U[NC];
#pragma unroll
    for (int v = 0; v < NC; ++v) U[v] = X[v * Nq + i];
    double r = U[0], ke = 0.0, vel[DIM];
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      vel[m] = U[1 + m] / r;
      ke += vel[m] * U[1 + m];
    }
    double p = gm1 * (U[DIM + 1] - 0.5 * ke);
    if (!(r > 0.0) || !(p > 0.0)) bad = 1;
    double s = log(p) - g * log(r), beta = r / p, v2 = 0.0;
#pragma unroll
    for (int m = 0; m < DIM; ++m) v2 += vel[m] * vel[m];
    double wj = gv[S::NG * Nq + i];
    X[0 * Nq + i] = wj * ((g - s) * gm1inv - 0.5 * beta * v2);
#pragma unroll
    for (int m = 0; m < DIM; ++m) X[(1 + m) * Nq + i] = wj * beta * vel[m];
    X[(DIM + 1) * Nq + i] = -wj * beta;
  }
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(T, X, um, T1, T2);
  modal_to_nodal<DIM, N, NC>(T, um, X, T1, T2);
  for (int it = tid; it < NC * Nq; it += nt) X[it] *= gv[(S::NG + 1) * Nq + it % Nq];  // W / J~
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(T, X, um, T1, T2);  // w~
  if (A.wt)
    for (int k = tid; k < NC * Np; k += nt) A.wt[(size_t)e * NC * Np + k] = um[k];
  modal_to_nodal<DIM, N, NC>(T, um, X, T1, T2);  // w = V w~
  // w_f = R^(z) w along lines
  for (int it = tid; it < NC * NF; it += nt) {
    int v = it / NF, fz = it % NF, z = fz / Nqf, f = fz % Nqf;
    const double* x = X + v * Nq;
    double s = 0.0;
    if constexpr (DIM == 2) {
      if (z == 0)
        for (int b = 0; b < N; ++b) s += __ldg(&R.lL[b]) * x[f + N * b];
      else
        for (int a = 0; a < N; ++a) s += __ldg(z == 1 ? &R.lR[a] : &R.lL[a]) * x[a + N * f];
    } else {
      int f1 = f % N, f2 = f / N;
      if (z == 0)
        for (int b = 0; b < N; ++b) s += __ldg(&R.lL[b]) * x[f1 + N * b + N * N * f2];
      else if (z < 3)
        for (int a = 0; a < N; ++a) s += __ldg(z == 1 ? &R.lR[a] : &R.lL[a]) * x[a + N * f1 + N * N * f2];
      else
        for (int c = 0; c < N; ++c) {
          double t = 0.0;
          for (int b = 0; b < N; ++b) t += __ldg(&R.lint4[f2 * N + b]) * x[f1 + N * b + N * N * c];
          s += __ldg(&R.l3L[c]) * t;
        }
    }
    FW[it] = s;
  }
  __syncthreads();
  // entropy-projected conservative variables U(w) -> stored as primitive (rho, v, p)
  auto Uofw = [&](const double* w, double* out) -> int {
    double b = -w[DIM + 1], vel[DIM], v2 = 0.0;
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      vel[m] = w[1 + m] / b;
      v2 += vel[m] * vel[m];
    }
    double s = g - gm1 * (w[0] + 0.5 * b * v2);
    double r = exp((s + log(b)) / (1.0 - g));
    out[0] = r;
#pragma unroll
    for (int m = 0; m < DIM; ++m) out[1 + m] = vel[m];
    out[DIM + 1] = r / b;
    return (b > 0.0 && r > 0.0) ? 0 : 1;
  };
  for (int i = tid; i < Nq; i += nt) {
    double w[NC], o[NC];
#pragma unroll
    for (int v = 0; v < NC; ++v) w[v] = X[v * Nq + i];
    bad |= Uofw(w, o);
#pragma unroll
    for (int v = 0; v < NC; ++v) A.prim[(size_t)e * S::PRS + v * Nq + i] = o[v];
  }
  for (int fz = tid; fz < NF; fz += nt) {
    double w[NC], o[NC];
#pragma unroll
    for (int v = 0; v < NC; ++v) w[v] = FW[v * NF + fz];
    bad |= Uofw(w, o);
    int z = fz / Nqf, f = fz % Nqf;
#pragma unroll
    for (int v = 0; v < NC; ++v) A.trace[(((size_t)e * S::Nf + z) * NC + v) * Nqf + f] = o[v];
  }
  if (bad) atomicOr(A.bad, 1);
}

// ------------------------------------------------------------------------------------------------
// nodal initial data -> modal: u~ = V^T W u  (R18)
// ------------------------------------------------------------------------------------------------
template <int DIM, int N>
__global__ void __launch_bounds__(Sz<DIM, N>::NT) project_nodal_kernel(DevRef R, int64_t ne, const double* un,
                                                                    double* um_out) {
  using S = Sz<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np;
  extern __shared__ double sm[];
  double* X = sm;
  double* um = X + NC * Nq;
  double* T1 = um + NC * Np;
  double* T2 = T1 + t1_size<DIM, N>();
  const PsiS T = stage_psi<DIM, N>(R, T2 + t2_size<DIM, N>());
  int64_t e = blockIdx.x;
  for (int it = threadIdx.x; it < NC * Nq; it += blockDim.x) {
    int v = it / Nq, i = it % Nq;
    X[it] = __ldg(&R.Wvol[i]) * un[((size_t)e * Nq + i) * NC + v];
  }
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(T, X, um, T1, T2);
  for (int k = threadIdx.x; k < NC * Np; k += blockDim.x) um_out[(size_t)e * NC * Np + k] = um[k];
}

template <int DIM, int N>
__host__ __device__ constexpr size_t projnodal_smem_doubles() {
  using S = Sz<DIM, N>;
  return (size_t)S::NC * S::Nq + (size_t)S::NC * S::Np + t1_size<DIM, N>() + t2_size<DIM, N>() +
         psi_smem_doubles<DIM, N>();
}

// host-side launchers (defined in kernels_2d.cu / kernels_3d.cu)
struct LaunchCfg {
  cudaStream_t stream;
};
cudaError_t launch_project(int dim, int n, const DevRef& R, const ProjArgs& A, cudaStream_t st);
cudaError_t launch_rhs(int dim, int n, const DevRef& R, const RhsArgs& A, cudaStream_t st);
cudaError_t launch_project_nodal(int dim, int n, const DevRef& R, int64_t ne, const double* un, double* um,
                                 cudaStream_t st);

}  // namespace esb
