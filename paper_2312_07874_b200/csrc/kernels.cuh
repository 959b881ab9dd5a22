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
  const double* geo_vol;     // [nloc][NGV][Nq]
  double* prim;              // [nloc][NC][Nq]   entropy-projected primitive (rho, v, p)
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
// sum-factorised PKD transforms, NV variables at once, block-wide
// ------------------------------------------------------------------------------------------------
template <int DIM, int N, int NV>
__device__ void modal_to_nodal(const DevRef& R, const double* um, double* un, double* t1, double* t2) {
  using S = Sz<DIM, N>;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (DIM == 2) {
    for (int it = tid; it < NV * N * N; it += nt) {  // t1[v][a1][b]
      int b = it % N, a1 = (it / N) % N, v = it / (N * N);
      int off = R.pair_off[a1];
      double s = 0.0;
      for (int a2 = 0; a2 <= S::P - a1; ++a2) s += __ldg(&R.psi2[(a1 * N + a2) * N + b]) * um[v * S::Np + off + a2];
      t1[it] = s;
    }
    __syncthreads();
    for (int it = tid; it < NV * S::Nq; it += nt) {
      int i = it % S::Nq, v = it / S::Nq, a = i % N, b = i / N;
      double s = 0.0;
#pragma unroll 4
      for (int a1 = 0; a1 < N; ++a1) s += __ldg(&R.psi1[a1 * N + a]) * t1[(v * N + a1) * N + b];
      un[it] = s;
    }
    __syncthreads();
  } else {
    for (int it = tid; it < NV * S::NPAIR * N; it += nt) {  // t1[v][pr][c]
      int c = it % N, pr = (it / N) % S::NPAIR, v = it / (N * S::NPAIR);
      int s = R.pair_a1[pr] + R.pair_a2[pr], off = R.pair_off[pr];
      double acc = 0.0;
      for (int a3 = 0; a3 <= S::P - s; ++a3) acc += __ldg(&R.psi3[(s * N + a3) * N + c]) * um[v * S::Np + off + a3];
      t1[it] = acc;
    }
    __syncthreads();
    for (int it = tid; it < NV * N * N * N; it += nt) {  // t2[v][a1][c][b]
      int b = it % N, c = (it / N) % N, a1 = (it / (N * N)) % N, v = it / (N * N * N);
      int prs = a1 * N - a1 * (a1 - 1) / 2;
      double acc = 0.0;
      for (int a2 = 0; a2 <= S::P - a1; ++a2)
        acc += __ldg(&R.psi2[(a1 * N + a2) * N + b]) * t1[(v * S::NPAIR + prs + a2) * N + c];
      t2[it] = acc;
    }
    __syncthreads();
    for (int it = tid; it < NV * S::Nq; it += nt) {
      int i = it % S::Nq, v = it / S::Nq, a = i % N, bc = i / N;
      double acc = 0.0;
#pragma unroll 4
      for (int a1 = 0; a1 < N; ++a1) acc += __ldg(&R.psi1[a1 * N + a]) * t2[(v * N + a1) * N * N + bc];
      un[it] = acc;
    }
    __syncthreads();
  }
}

template <int DIM, int N, int NV>
__device__ void nodal_to_modal(const DevRef& R, const double* y, double* um, double* t1, double* t2) {
  using S = Sz<DIM, N>;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (DIM == 2) {
    for (int it = tid; it < NV * N * N; it += nt) {  // s1[v][a1][b]
      int b = it % N, a1 = (it / N) % N, v = it / (N * N);
      double s = 0.0;
#pragma unroll 4
      for (int a = 0; a < N; ++a) s += __ldg(&R.psi1[a1 * N + a]) * y[v * S::Nq + a + N * b];
      t1[it] = s;
    }
    __syncthreads();
    for (int it = tid; it < NV * S::Np; it += nt) {
      int k = it % S::Np, v = it / S::Np;
      int a1 = R.mode_pr[k], a2 = R.mode_last[k];
      double s = 0.0;
#pragma unroll 4
      for (int b = 0; b < N; ++b) s += __ldg(&R.psi2[(a1 * N + a2) * N + b]) * t1[(v * N + a1) * N + b];
      um[it] = s;
    }
    __syncthreads();
  } else {
    for (int it = tid; it < NV * N * N * N; it += nt) {  // s2[v][a1][b][c]
      int bc = it % (N * N), a1 = (it / (N * N)) % N, v = it / (N * N * N);
      double acc = 0.0;
#pragma unroll 4
      for (int a = 0; a < N; ++a) acc += __ldg(&R.psi1[a1 * N + a]) * y[v * S::Nq + a + N * bc];
      t2[it] = acc;
    }
    __syncthreads();
    for (int it = tid; it < NV * S::NPAIR * N; it += nt) {  // s1[v][pr][c]
      int c = it % N, pr = (it / N) % S::NPAIR, v = it / (N * S::NPAIR);
      int a1 = R.pair_a1[pr], a2 = R.pair_a2[pr];
      double acc = 0.0;
#pragma unroll 4
      for (int b = 0; b < N; ++b)
        acc += __ldg(&R.psi2[(a1 * N + a2) * N + b]) * t2[((v * N + a1) * N + c) * N + b];
      t1[it] = acc;
    }
    __syncthreads();
    for (int it = tid; it < NV * S::Np; it += nt) {
      int k = it % S::Np, v = it / S::Np;
      int pr = R.mode_pr[k], a3 = R.mode_last[k];
      int s = R.pair_a1[pr] + R.pair_a2[pr];
      double acc = 0.0;
#pragma unroll 4
      for (int c = 0; c < N; ++c) acc += __ldg(&R.psi3[(s * N + a3) * N + c]) * t1[(v * S::NPAIR + pr) * N + c];
      um[it] = acc;
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
         (size_t)S::NC * S::NF;
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
  const int64_t e = A.elem_list ? A.elem_list[blockIdx.x] : (int64_t)blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double g = A.gamma, gm1 = g - 1.0, gm1inv = 1.0 / gm1;
  const double* gv = A.geo_vol + (size_t)e * S::NGV * Nq;
  for (int k = tid; k < NC * Np; k += nt) um[k] = A.u[(size_t)e * NC * Np + k];
  __syncthreads();
  modal_to_nodal<DIM, N, NC>(R, um, X, T1, T2);  // u = V u~
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
  nodal_to_modal<DIM, N, NC>(R, X, um, T1, T2);
  modal_to_nodal<DIM, N, NC>(R, um, X, T1, T2);
  for (int it = tid; it < NC * Nq; it += nt) X[it] *= gv[(S::NG + 1) * Nq + it % Nq];  // W / J~
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(R, X, um, T1, T2);  // w~
  if (A.wt)
    for (int k = tid; k < NC * Np; k += nt) A.wt[(size_t)e * NC * Np + k] = um[k];
  modal_to_nodal<DIM, N, NC>(R, um, X, T1, T2);  // w = V w~
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
    for (int v = 0; v < NC; ++v) A.prim[((size_t)e * NC + v) * Nq + i] = o[v];
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
// K2: flux differencing + facet correction + interface + lifting + weight-adjusted inverse
// ------------------------------------------------------------------------------------------------
template <int DIM, int N>
struct RhsSmem {
  using S = Sz<DIM, N>;
  static constexpr int PR = (DIM + 3) * S::Nq;  // rho, v, p, beta
  static constexpr int GG = S::NG * S::Nq;
  static constexpr int XB = S::NC * S::Nq;
  static constexpr int FP = S::NC * S::NF;
  static constexpr int FJ = DIM * S::NF;
  static constexpr int CT = S::NC * S::NF;
  static constexpr int PT = S::NC * N * N;
  static constexpr int TB = 5 * N * N + 6 * N + N * N + S::NF;
  static constexpr int o_pr = 0, o_g = o_pr + PR, o_xb = o_g + GG, o_fp = o_xb + XB, o_fj = o_fp + FP,
                       o_ct = o_fj + FJ, o_pt = o_ct + CT, o_tb = o_pt + PT, total = o_tb + TB;
  static_assert(t1_size<DIM, N>() + t2_size<DIM, N>() <= PR + GG, "transform scratch");
  static_assert(S::NC * S::Np <= FP + FJ + CT + PT, "modal scratch");
};

template <int DIM, int N>
__host__ __device__ constexpr size_t rhs_smem_doubles() {
  return RhsSmem<DIM, N>::total;
}

template <int DIM, int N>
__global__ void __launch_bounds__(Sz<DIM, N>::NT) rhs_kernel(DevRef R, RhsArgs A) {
  using S = Sz<DIM, N>;
  using L = RhsSmem<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf, NT = S::NT, KPT = S::KPT;
  extern __shared__ double sm[];
  double* sP = sm + L::o_pr;   // [DIM+3][Nq]: rho, v_1..v_d, p, beta
  double* sG = sm + L::o_g;    // [NG][Nq]: G_lm at (l*DIM+m)
  double* xb = sm + L::o_xb;   // [NC][Nq] exchange buffer / nodal residual
  double* fP = sm + L::o_fp;   // [NC][NF] own facet states (rho, v, p)
  double* fJ = sm + L::o_fj;   // [DIM][NF] J n
  double* ct = sm + L::o_ct;   // [NC][NF] C^T 1, then s = B J_f f* - C^T 1
  double* pt = sm + L::o_pt;   // [NC][N][N] facet-4 partial sums
  double* tb = sm + L::o_tb;   // tables
  double* tQ1 = tb;
  double* tA1 = tQ1 + N * N;
  double* tA2 = tA1 + N * N;
  double* tA3 = tA2 + N * N;
  double* tA4 = tA3 + N * N;
  double* tw = tA4 + N * N;
  double* tw3 = tw + N;
  double* teta = tw3 + N;
  double* tlL = teta + N;
  double* tlR = tlL + N;
  double* tl3 = tlR + N;
  double* tli4 = tl3 + N;
  double* tB = tli4 + N * N;

  const int64_t e = A.elem_list ? A.elem_list[blockIdx.x] : (int64_t)blockIdx.x;
  const int tid = threadIdx.x;
  const double g = A.gamma, gm1inv = 1.0 / (g - 1.0);
  // ---- stage tables, states and metrics in shared memory ----
  for (int k = tid; k < N * N; k += NT) {
    tQ1[k] = R.skQ1[k];
    tA1[k] = R.skA1[k];
    tA2[k] = R.skA2[k];
    if constexpr (DIM == 3) {
      tA3[k] = R.skA3[k];
      tA4[k] = R.skA4[k];
    }
    tli4[k] = DIM == 3 ? R.lint4[k] : 0.0;
  }
  for (int k = tid; k < N; k += NT) {
    tw[k] = R.w[k];
    tw3[k] = R.w3[k];
    teta[k] = R.eta[k];
    tlL[k] = R.lL[k];
    tlR[k] = R.lR[k];
    tl3[k] = DIM == 3 ? R.l3L[k] : 0.0;
  }
  for (int k = tid; k < NF; k += NT) tB[k] = R.Bf[k];
  const double* pe = A.prim + (size_t)e * NC * Nq;
  for (int k = tid; k < NC * Nq; k += NT) sP[k] = pe[k];
  const double* gv = A.geo_vol + (size_t)e * S::NGV * Nq;
  for (int k = tid; k < S::NG * Nq; k += NT) sG[k] = gv[k];
  for (int k = tid; k < NC * NF; k += NT) {
    int v = k / NF, fz = k % NF;
    fP[k] = A.trace[(((size_t)e * S::Nf + fz / Nqf) * NC + v) * Nqf + fz % Nqf];
    ct[k] = 0.0;
  }
  const double* gf = A.geo_face + (size_t)e * S::Nf * DIM * Nqf;
  for (int k = tid; k < DIM * NF; k += NT) {
    int m = (k / Nqf) % DIM, z = k / (DIM * Nqf), f = k % Nqf;
    fJ[m * NF + z * Nqf + f] = gf[k];
  }
  __syncthreads();
  for (int i = tid; i < Nq; i += NT) sP[(DIM + 2) * Nq + i] = sP[i] / sP[(DIM + 1) * Nq + i];  // beta
  __syncthreads();

  double acc[KPT][NC];
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk)
#pragma unroll
    for (int v = 0; v < NC; ++v) acc[kk][v] = 0.0;

  auto load_state = [&](int i, double& r, double* vel, double& p, double& b) {
    r = sP[i];
#pragma unroll
    for (int m = 0; m < DIM; ++m) vel[m] = sP[(1 + m) * Nq + i];
    p = sP[(DIM + 1) * Nq + i];
    b = sP[(DIM + 2) * Nq + i];
  };
  auto Gat = [&](int l, int m, int i) { return sG[(l * DIM + m) * Nq + i]; };

  // ---- volume terms: one EC flux per node pair on every eta_k line ----
#pragma unroll 1
  for (int k = 0; k < DIM; ++k) {
    const int stride = k == 0 ? 1 : (k == 1 ? N : N * N);
#pragma unroll 1
    for (int s = 1; s <= N / 2; ++s) {
      const bool half = (N % 2 == 0) && (s == N / 2);
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) {
        int i = tid + kk * NT;
        if (i >= Nq) break;
        int a = i % N, b = (i / N) % N, c = DIM == 3 ? i / (N * N) : 0;
        int pos = k == 0 ? a : (k == 1 ? b : c);
        if (half && pos >= N / 2) continue;
        int pos2 = pos + s;
        if (pos2 >= N) pos2 -= N;
        int j = i + (pos2 - pos) * stride;
        double nv[DIM];
        const int ix = pos * N + pos2;
        if constexpr (DIM == 2) {
          if (k == 0) {
            double cl = tw[b], q1 = tQ1[ix], a1 = tA1[ix];
#pragma unroll
            for (int m = 0; m < DIM; ++m)
              nv[m] = cl * (q1 * (Gat(0, m, i) + Gat(0, m, j)) + a1 * (Gat(1, m, i) + Gat(1, m, j)));
          } else {
            double cl = tw[a] * tA2[ix];
#pragma unroll
            for (int m = 0; m < DIM; ++m) nv[m] = cl * (Gat(1, m, i) + Gat(1, m, j));
          }
        } else {
          if (k == 0) {
            double cl = 0.5 * tw[b] * tw3[c], q1 = tQ1[ix], a1 = tA1[ix];
#pragma unroll
            for (int m = 0; m < DIM; ++m)
              nv[m] = cl * (q1 * (Gat(0, m, i) + Gat(0, m, j)) +
                            a1 * (Gat(1, m, i) + Gat(2, m, i) + Gat(1, m, j) + Gat(2, m, j)));
          } else if (k == 1) {
            double cl = 0.5 * tw[a] * tw3[c], a2 = tA2[ix], a3 = tA3[ix];
#pragma unroll
            for (int m = 0; m < DIM; ++m)
              nv[m] = cl * (a2 * (Gat(1, m, i) + Gat(1, m, j)) + a3 * (Gat(2, m, i) + Gat(2, m, j)));
          } else {
            double cl = 0.125 * tw[a] * tw[b] * (1.0 - teta[b]) * tA4[ix];
#pragma unroll
            for (int m = 0; m < DIM; ++m) nv[m] = cl * (Gat(2, m, i) + Gat(2, m, j));
          }
        }
        double ri, vi[DIM], pi_, bi, rj, vj[DIM], pj, bj, F[NC];
        load_state(i, ri, vi, pi_, bi);
        load_state(j, rj, vj, pj, bj);
        ec_flux<DIM>(ri, vi, pi_, bi, rj, vj, pj, bj, nv, gm1inv, F);
#pragma unroll
        for (int v = 0; v < NC; ++v) {
          acc[kk][v] -= F[v];
          xb[v * Nq + i] = F[v];
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) {
        int i = tid + kk * NT;
        if (i >= Nq) break;
        int a = i % N, b = (i / N) % N, c = DIM == 3 ? i / (N * N) : 0;
        int pos = k == 0 ? a : (k == 1 ? b : c);
        if (half && pos < N / 2) continue;
        int pos0 = pos - s;
        if (pos0 < 0) pos0 += N;
        int i0 = i + (pos0 - pos) * stride;
#pragma unroll
        for (int v = 0; v < NC; ++v) acc[kk][v] += xb[v * Nq + i0];
      }
      __syncthreads();
    }
  }

  // ---- facet correction C: volume node i with facet node f ----
  auto facet_pair = [&](int i, int z, int f, double coef, int kk) {
    double nv[DIM];
#pragma unroll
    for (int m = 0; m < DIM; ++m) {  // <J n>_if = (G_i^T nhat + G_f^T nhat)/2
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < DIM; ++l) s += Gat(l, m, i) * __ldg(&R.nhat[z * 3 + l]);
      nv[m] = 0.5 * (s + fJ[m * NF + z * Nqf + f]);
    }
    double ri, vi[DIM], pi_, bi, F[NC];
    load_state(i, ri, vi, pi_, bi);
    int fz = z * Nqf + f;
    double rf = fP[fz], vf[DIM], pf;
#pragma unroll
    for (int m = 0; m < DIM; ++m) vf[m] = fP[(1 + m) * NF + fz];
    pf = fP[(DIM + 1) * NF + fz];
    ec_flux<DIM>(ri, vi, pi_, bi, rf, vf, pf, rf / pf, nv, gm1inv, F);
#pragma unroll
    for (int v = 0; v < NC; ++v) {
      double c = coef * F[v];
      acc[kk][v] -= c;
      xb[v * Nq + i] = c;
    }
  };
#pragma unroll 1
  for (int z = 0; z < 3; ++z) {  // facets whose extrapolation acts along one line
#pragma unroll
    for (int kk = 0; kk < KPT; ++kk) {
      int i = tid + kk * NT;
      if (i >= Nq) break;
      int a = i % N, b = (i / N) % N, c = DIM == 3 ? i / (N * N) : 0;
      int f;
      double coef;
      if (z == 0) {  // eta2 = -1
        f = DIM == 2 ? a : a + N * c;
        coef = tlL[b];
      } else {  // eta1 = +1 / -1
        f = DIM == 2 ? b : b + N * c;
        coef = z == 1 ? tlR[a] : tlL[a];
      }
      facet_pair(i, z, f, coef * tB[z * Nqf + f], kk);
    }
    __syncthreads();
    for (int it = tid; it < NC * Nqf; it += NT) {  // C^T 1 on facet z: sum along the line
      int v = it / Nqf, f = it % Nqf;
      double s = 0.0;
      if (z == 0) {
        int a = DIM == 2 ? f : f % N, c = DIM == 2 ? 0 : f / N;
        for (int b = 0; b < N; ++b) s += xb[v * Nq + a + N * b + N * N * c];
      } else {
        for (int a = 0; a < N; ++a) s += xb[v * Nq + a + N * f];
      }
      ct[v * NF + z * Nqf + f] = s;
    }
    __syncthreads();
  }
  if constexpr (DIM == 3) {  // facet 4 (eta3 = -1): couples the whole (eta2, eta3) plane
#pragma unroll 1
    for (int jf = 0; jf < N; ++jf) {
#pragma unroll
      for (int kk = 0; kk < KPT; ++kk) {
        int i = tid + kk * NT;
        if (i >= Nq) break;
        int a = i % N, b = (i / N) % N, c = i / (N * N);
        int f = a + N * jf;
        facet_pair(i, 3, f, tli4[jf * N + b] * tl3[c] * tB[3 * Nqf + f], kk);
      }
      __syncthreads();
      for (int it = tid; it < NC * N * N; it += NT) {  // partial sums over b
        int v = it / (N * N), a = (it / N) % N, c = it % N;
        double s = 0.0;
        for (int b = 0; b < N; ++b) s += xb[v * Nq + a + N * b + N * N * c];
        pt[(v * N + a) * N + c] = s;
      }
      __syncthreads();
      for (int it = tid; it < NC * N; it += NT) {
        int v = it / N, a = it % N;
        double s = 0.0;
        for (int c = 0; c < N; ++c) s += pt[(v * N + a) * N + c];
        ct[v * NF + 3 * Nqf + a + N * jf] = s;
      }
      // (the next iteration's first barrier orders these reads before pt is rewritten)
    }
    __syncthreads();
  }

  // ---- interface flux and s = B J_f f* - C^T 1 ----
  for (int fz = tid; fz < NF; fz += NT) {
    int z = fz / Nqf, f = fz % Nqf;
    int64_t slot = A.face_slot[e * S::Nf + z];
    int rf = A.face_reflect[e * S::Nf + z];
    int fo;
    if constexpr (DIM == 2)
      fo = rf ? N - 1 - f : f;
    else
      fo = rf ? (N - 1 - f % N) + N * (f / N) : f;
    const double* tp = A.trace + (size_t)slot * NC * Nqf;
    double rp = tp[fo], vp[DIM], pp;
#pragma unroll
    for (int m = 0; m < DIM; ++m) vp[m] = tp[(1 + m) * Nqf + fo];
    pp = tp[(DIM + 1) * Nqf + fo];
    double rm = fP[fz], vm[DIM], pm;
#pragma unroll
    for (int m = 0; m < DIM; ++m) vm[m] = fP[(1 + m) * NF + fz];
    pm = fP[(DIM + 1) * NF + fz];
    double Jn[DIM], Jf = 0.0;
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      Jn[m] = fJ[m * NF + fz];
      Jf += Jn[m] * Jn[m];
    }
    Jf = sqrt(Jf);
    double nu[DIM];
#pragma unroll
    for (int m = 0; m < DIM; ++m) nu[m] = Jn[m] / Jf;
    double F[NC];
    ec_flux<DIM>(rm, vm, pm, rm / pm, rp, vp, pp, rp / pp, nu, gm1inv, F);
    if (A.es) {  // local Lax-Friedrichs with Davis's wave speed
      double vnm = 0.0, vnp = 0.0;
#pragma unroll
      for (int m = 0; m < DIM; ++m) {
        vnm += vm[m] * nu[m];
        vnp += vp[m] * nu[m];
      }
      double lam = fmax(fabs(vnm), fabs(vnp)) + fmax(sqrt(g * pm / rm), sqrt(g * pp / rp));
      double Um[NC], Up[NC];
      cons_of<DIM>(rm, vm, pm, gm1inv, Um);
      cons_of<DIM>(rp, vp, pp, gm1inv, Up);
#pragma unroll
      for (int v = 0; v < NC; ++v) F[v] -= 0.5 * lam * (Up[v] - Um[v]);
    }
    double bj = tB[fz] * Jf;
#pragma unroll
    for (int v = 0; v < NC; ++v) ct[v * NF + fz] = bj * F[v] - ct[v * NF + fz];
  }
  __syncthreads();

  // ---- lifting r -= R^T s and residual to shared memory ----
#pragma unroll
  for (int kk = 0; kk < KPT; ++kk) {
    int i = tid + kk * NT;
    if (i >= Nq) break;
    int a = i % N, b = (i / N) % N, c = DIM == 3 ? i / (N * N) : 0;
#pragma unroll
    for (int v = 0; v < NC; ++v) {
      const double* sv = ct + v * NF;
      double t;
      if constexpr (DIM == 2) {
        t = tlL[b] * sv[a] + tlR[a] * sv[Nqf + b] + tlL[a] * sv[2 * Nqf + b];
      } else {
        t = tlL[b] * sv[a + N * c] + tlR[a] * sv[Nqf + b + N * c] + tlL[a] * sv[2 * Nqf + b + N * c];
        double t4 = 0.0;
        for (int jf = 0; jf < N; ++jf) t4 += tli4[jf * N + b] * sv[3 * Nqf + a + N * jf];
        t += tl3[c] * t4;
      }
      xb[v * Nq + i] = acc[kk][v] - t;
    }
  }
  __syncthreads();

  // ---- d u~/dt = V^T W/J~ V (V^T r) ----
  double* T1 = sm + L::o_pr;
  double* T2 = T1 + t1_size<DIM, N>();
  double* um = sm + L::o_fp;
  nodal_to_modal<DIM, N, NC>(R, xb, um, T1, T2);
  if (A.mode == 5) {  // entropy production sum w~ . (V^T r) and conservation (V^T r)_0 / c0
    double loc = 0.0, la = 0.0;
    for (int k = tid; k < NC * Np; k += NT) {
      double t = A.wt[(size_t)e * NC * Np + k] * um[k];
      loc += t;
      la += fabs(t);
    }
    for (int o = 16; o > 0; o >>= 1) {
      loc += __shfl_down_sync(0xffffffffu, loc, o);
      la += __shfl_down_sync(0xffffffffu, la, o);
    }
    __shared__ double red[2][NT / 32];
    if ((tid & 31) == 0) {
      red[0][tid / 32] = loc;
      red[1][tid / 32] = la;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int wv = 0; wv < NT / 32; ++wv) {
        s0 += red[0][wv];
        s1 += red[1][wv];
      }
      double* pe2 = A.part + (size_t)e * (2 + NC);
      pe2[0] = s0;
      pe2[1] = s1;
      for (int v = 0; v < NC; ++v) pe2[2 + v] = um[v * Np] / A.c0;
    }
  }
  modal_to_nodal<DIM, N, NC>(R, um, xb, T1, T2);
  for (int it = tid; it < NC * Nq; it += NT) xb[it] *= gv[(S::NG + 1) * Nq + it % Nq];
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(R, xb, um, T1, T2);
  const size_t base = (size_t)e * NC * Np;
  const double dt = A.dt;
  for (int k = tid; k < NC * Np; k += NT) {
    double du = um[k];
    switch (A.mode) {
      case 0:
      case 5:
        A.out[base + k] = du;
        break;
      case 1:  // classical RK4 stage 1 (R17)
        A.acc[base + k] = A.u0[base + k] + (dt / 6.0) * du;
        A.ustage[base + k] = A.u0[base + k] + (0.5 * dt) * du;
        break;
      case 2:
        A.acc[base + k] += (dt / 3.0) * du;
        A.ustage[base + k] = A.u0[base + k] + (0.5 * dt) * du;
        break;
      case 3:
        A.acc[base + k] += (dt / 3.0) * du;
        A.ustage[base + k] = A.u0[base + k] + dt * du;
        break;
      case 4:
        A.out[base + k] = A.acc[base + k] + (dt / 6.0) * du;  // out = new state
        break;
    }
  }
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
  int64_t e = blockIdx.x;
  for (int it = threadIdx.x; it < NC * Nq; it += blockDim.x) {
    int v = it / Nq, i = it % Nq;
    X[it] = __ldg(&R.Wvol[i]) * un[((size_t)e * Nq + i) * NC + v];
  }
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(R, X, um, T1, T2);
  for (int k = threadIdx.x; k < NC * Np; k += blockDim.x) um_out[(size_t)e * NC * Np + k] = um[k];
}

template <int DIM, int N>
__host__ __device__ constexpr size_t projnodal_smem_doubles() {
  using S = Sz<DIM, N>;
  return (size_t)S::NC * S::Nq + (size_t)S::NC * S::Np + t1_size<DIM, N>() + t2_size<DIM, N>();
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
