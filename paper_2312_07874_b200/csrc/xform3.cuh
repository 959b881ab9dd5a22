// xform3.cuh -- K3 (tetrahedra): the weight-adjusted inverse mass matrix
//     du~/dt = V^T diag(W / J~) V (V^T r)
// on the nodal residual r written by the flux kernel, batched over E elements per CTA, with the
// classical RK4 stage update / entropy-production partials fused into the epilogue.  Product code.
//
// Sum factorisation over the collapsed coordinates:
//   V:   t1[pr][c] = sum_a3 psi3[s][a3][c] u~[pr][a3]          (s = a1 + a2, pr = (a1, a2))
//        t2[a1][b] = sum_a2 psi2[a1][a2][b] t1[pr(a1, a2)]      (for each c)
//        u[a][b]   = sum_a1 psi1[a1][a] t2[a1][b]                (for each c)
//   V^T: the same three contractions transposed, in reverse order.
// Two lane mappings alternate, each chosen so that the PKD tables are warp-uniform -- they are read
// from constant memory as uniform-register operands of DFMA, never from shared memory:
//   mode A, lane = (element, variable, c): the psi1 / psi2 contractions of one c-slab run entirely in
//        registers (the psi3 index c is the lane's own), e.g. V^T steps 1-2, or V steps 2-3 followed by
//        the W / J~ scaling and V^T steps 1-2 with nothing but the c-slab's 45 t1 values in between;
//   mode B, lane = (pr, element, variable), lanes ordered by pr sorted on s so that a warp shares one
//        pr: the psi3 contraction of one (pr) fibre over c, specialised at compile time on its length
//        N - s (V^T step 3, then V step 1 of the next transform in the same registers).
// Between the modes the (pr, c) slabs go through shared memory S[e][v][pr][c] (one barrier each).
// Global layouts chosen for coalescing in mode A (c fastest): the residual r[e][v][b][a][c] (written
// so by the flux kernel) and W / J~ [e][b][a][c] (permuted copy made at setup).
#pragma once
#include "kernels.cuh"
#include "psi_const.cuh"

namespace esb {

template <int N>
struct X3 {
  static constexpr int NPAIR = N * (N + 1) / 2, Np = N * (N + 1) * (N + 2) / 6, Nq = N * N * N, NC = 5;
  // S stride per (element, variable) = N (mod 16) doubles: the N-lane groups of a warp then tile the
  // shared-memory banks two deep (mode A) and B-mode lanes hit distinct bank pairs
  static constexpr int SEV = NPAIR * N + ((N - NPAIR * N) % 16 + 16) % 16;
  static constexpr int SPE = NC * SEV;  // S doubles per element: [v][pr][c] (+ pad)
  static constexpr int UPE = NC * Np;  // modal result [v][k] (the element's W / J~ [b][a][c] before that)
  static_assert(NC * Np >= Nq, "W / J~ staging fits the modal buffer");
  static constexpr int PPE = NC * (2 * NPAIR + 1);  // entropy partials per element
  // elements per CTA: the mode-A lanes (5 E N) fill whole warps of a CTA of at most 192 threads
  // (two CTAs per SM, so that one CTA's global loads and barriers overlap the other's arithmetic)
#ifndef ES_K3_THREADS
#define ES_K3_THREADS 192
#endif
#ifndef ES_K3_MINB
#define ES_K3_MINB 2
#endif
  static constexpr int MINB = ES_K3_MINB;  // resident CTAs per SM the register budget is sized for
  static constexpr int E = (ES_K3_THREADS / (NC * N)) < 1 ? 1 : (ES_K3_THREADS / (NC * N));
  static constexpr int NT = ((NC * E * N + 31) / 32) * 32;
  static constexpr size_t SMEM = (size_t)E * (SPE + UPE + PPE) * sizeof(double);
};

// pair index and modal offset of (a1, a2) in the alpha1-major nested order (R9)
__host__ __device__ constexpr int pr_of(int N, int a1, int a2) { return a1 * N - a1 * (a1 - 1) / 2 + a2; }
__host__ __device__ constexpr int off_of(int N, int a1, int a2) {
  int o = 0;
  for (int x1 = 0; x1 < a1; ++x1)
    for (int x2 = 0; x2 < N - x1; ++x2) o += N - x1 - x2;
  for (int x2 = 0; x2 < a2; ++x2) o += N - a1 - x2;
  return o;
}

struct WadjArgs {
  int64_t n_elem;
  const double* r;      // [n][NC][N(b)][N(a)][N(c)] nodal residual (flux kernel output)
  const double* wjinv;  // [n][N(b)][N(a)][N(c)] W / J~
  int mode;             // 0 dudt, 1..4 RK stage 0..3, 5 dudt + entropy partials
  double* out;
  const double* u0;
  double* acc;
  double* ustage;
  double dt;
  const double* wt;  // entropy mode: w~ [n][NC][Np]
  double* part;      // entropy mode: [n][2 + NC]
  double c0;
};

// ---- mode A: one c-slab, lane = (element, variable, c) ----
// Fully unrolled: every table read is a compile-time constant-memory operand (uniform registers).
// V^T steps 1-2 from the global residual: s1[pr] = sum_b psi2[a1][a2][b] sum_a psi1[a1][a] r[b][a][c]
template <int N>
__device__ __forceinline__ void modeA_vt12_global(const double* __restrict__ rr, double* S, bool ok, bool act) {
  constexpr int NPAIR = X3<N>::NPAIR;
  double s1[NPAIR];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) s1[q] = 0.0;
#pragma unroll
  for (int b = 0; b < N; ++b) {
    double x[N], s2[N];
#pragma unroll
    for (int a = 0; a < N; ++a) x[a] = ok ? __ldg(rr + (b * N + a) * N) : 0.0;
    psi1T_apply_eo<N>(x, s2);
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1)
#pragma unroll
      for (int a2 = 0; a2 < N - a1; ++a2)
        s1[pr_of(N, a1, a2)] = fma(c_psi<N>.p2[(a1 * N + a2) * N + b], s2[a1], s1[pr_of(N, a1, a2)]);
  }
  if (act)
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) S[q * N] = s1[q];
}

// V steps 2-3 of one c-slab, W / J~ scaling, V^T steps 1-2: S (t1 in) -> S (s1 out), same slots;
// wj: the element's W / J~ [b][a][c] in shared memory at the lane's c.  The t1 column is re-read
// from shared memory for every b (volatile: not hoisted into 2 x 45 registers beside the 45
// accumulators s1)
template <int N>
__device__ __forceinline__ void modeA_mid(double* S, const double* wj, bool act) {
  constexpr int NPAIR = X3<N>::NPAIR;
  const volatile double* Sv = S;
  double s1[NPAIR];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) s1[q] = 0.0;
#pragma unroll
  for (int b = 0; b < N; ++b) {
    double t2[N], y[N], s2[N];
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1) {
      double t = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < N - a1; ++a2) t = fma(c_psi<N>.p2[(a1 * N + a2) * N + b], Sv[pr_of(N, a1, a2) * N], t);
      t2[a1] = t;
    }
    psi1_apply_eo<N>(t2, y);
#pragma unroll
    for (int a = 0; a < N; ++a) y[a] *= wj[(b * N + a) * N];
    psi1T_apply_eo<N>(y, s2);
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1)
#pragma unroll
      for (int a2 = 0; a2 < N - a1; ++a2)
        s1[pr_of(N, a1, a2)] = fma(c_psi<N>.p2[(a1 * N + a2) * N + b], s2[a1], s1[pr_of(N, a1, a2)]);
  }
  if (act)
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) S[q * N] = s1[q];
}

// modeA_mid with the t1 column held in registers (45 loads per lane instead of 45 per b): 90
// accumulator + t1 doubles live, for CTAs sized to 1 per SM with a 224-register budget
template <int N>
__device__ __forceinline__ void modeA_mid_t1reg(double* S, const double* wj, bool act) {
  constexpr int NPAIR = X3<N>::NPAIR;
  double s1[NPAIR], t1[NPAIR];
#pragma unroll
  for (int q = 0; q < NPAIR; ++q) {
    s1[q] = 0.0;
    t1[q] = S[q * N];
  }
#pragma unroll
  for (int b = 0; b < N; ++b) {
    double t2[N], y[N], s2[N];
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1) {
      double t = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < N - a1; ++a2) t = fma(c_psi<N>.p2[(a1 * N + a2) * N + b], t1[pr_of(N, a1, a2)], t);
      t2[a1] = t;
    }
    psi1_apply_eo<N>(t2, y);
#pragma unroll
    for (int a = 0; a < N; ++a) y[a] *= wj[(b * N + a) * N];
    psi1T_apply_eo<N>(y, s2);
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1)
#pragma unroll
      for (int a2 = 0; a2 < N - a1; ++a2)
        s1[pr_of(N, a1, a2)] = fma(c_psi<N>.p2[(a1 * N + a2) * N + b], s2[a1], s1[pr_of(N, a1, a2)]);
  }
  if (act)
#pragma unroll
    for (int q = 0; q < NPAIR; ++q) S[q * N] = s1[q];
}

// ---- mode B: one (pr) fibre over c, length N3 = N - s of the modal index a3 ----
// V^T step 3 (u1[a3] = sum_c psi3[s][a3][c] x[c]) then, for FWD, V step 1 back into x (in place)
template <int N, int N3, bool FWD>
__device__ __forceinline__ void modeB_fibre(double* Sx, double* um, double& ent, double& ent_abs,
                                            const double* __restrict__ wt) {
  constexpr int s = N - N3;
  double x[N], u1[N3];
#pragma unroll
  for (int c = 0; c < N; ++c) x[c] = Sx[c];
#pragma unroll
  for (int a3 = 0; a3 < N3; ++a3) {
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < N; ++c) t = fma(c_psi<N>.p3[(s * N + a3) * N + c], x[c], t);
    u1[a3] = t;
  }
  if (wt) {  // entropy production: w~ . (V^T r)
#pragma unroll
    for (int a3 = 0; a3 < N3; ++a3) {
      const double t = __ldg(wt + a3) * u1[a3];
      ent += t;
      ent_abs += fabs(t);
    }
  }
  if constexpr (FWD) {
#pragma unroll
    for (int c = 0; c < N; ++c) {
      double t = 0.0;
#pragma unroll
      for (int a3 = 0; a3 < N3; ++a3) t = fma(c_psi<N>.p3[(s * N + a3) * N + c], u1[a3], t);
      Sx[c] = t;
    }
    if (um) um[0] = u1[0];  // the constant mode of V^T r (conservation), pr = 0 only
  } else {
#pragma unroll
    for (int a3 = 0; a3 < N3; ++a3) um[a3] = u1[a3];
  }
}

template <int N, bool FWD>
__device__ __forceinline__ void modeB_dispatch(int n3, double* Sx, double* um, double& ent, double& ent_abs,
                                               const double* wt) {
  switch (n3) {
#define ES_B_CASE(K) \
  case K:            \
    if constexpr (K <= N) modeB_fibre<N, (K <= N ? K : 1), FWD>(Sx, um, ent, ent_abs, wt); \
    break;
    ES_B_CASE(1) ES_B_CASE(2) ES_B_CASE(3) ES_B_CASE(4) ES_B_CASE(5) ES_B_CASE(6) ES_B_CASE(7) ES_B_CASE(8)
    ES_B_CASE(9) ES_B_CASE(10) ES_B_CASE(11)
#undef ES_B_CASE
    default: break;
  }
}

// B-mode pair ranks sorted by s = a1 + a2 (so that a warp shares one pr): rank -> (a1, a2)
template <int N>
__device__ __forceinline__ void pr_by_rank(int rank, int& a1, int& a2) {
  int s = 0, base = 0;
  while (rank >= base + s + 1) {
    base += s + 1;
    ++s;
  }
  a1 = rank - base;
  a2 = s - a1;
}

template <int N>
__global__ void __launch_bounds__(X3<N>::NT, X3<N>::MINB) wadj3_kernel(const WadjArgs A) {
  pdl_wait();
  PDL_TRIGGER();
  using Z = X3<N>;
  constexpr int NC = Z::NC, NPAIR = Z::NPAIR, Np = Z::Np, E = Z::E, NT = Z::NT, SPE = Z::SPE, UPE = Z::UPE;
  extern __shared__ __align__(16) double smx[];
  double* S = smx;            // [E][NC][NPAIR][N]
  double* U = smx + E * SPE;  // [E][NC][Np] modal result, then the entropy partials
  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * E;
  const int ne = (int)((A.n_elem - e0) < E ? (A.n_elem - e0) : E);
  const bool ent_mode = A.mode == 5;
  // W / J~ of the CTA's elements into the (not yet used) modal buffer U[e] ([b][a][c], 8-byte
  // asynchronous copies: the element stride of U is odd), consumed by A2
  for (int k = tid; k < ne * Z::Nq; k += NT) {
    const int e = k / Z::Nq, q = k - e * Z::Nq;
    cp_async8(U + e * UPE + q, A.wjinv + (e0 + e) * Z::Nq + q);
  }
  cp_async_commit();

  // ---- A1: V^T steps 1-2 of r, lane = (e, v, c); every thread runs it (warp-convergent, so that the
  // b-dependent table rows are uniform-register constant loads), idle lanes on zeros without stores
  {
    const bool act = tid < NC * E * N;
    const int ev = act ? tid / N : 0, c = act ? tid - ev * N : 0, e = ev / NC;
    const bool ok = act && e < ne;
    modeA_vt12_global<N>(A.r + ((size_t)e0 * NC + (ok ? ev : 0)) * Z::Nq + c, S + ev * Z::SEV + c, ok, act);
  }
  __syncthreads();
  // ---- B1: V^T step 3 (r^ = V^T r) and V step 1, lane = (pr rank, e, v) ----
  double* pe = U + E * UPE;  // entropy partials [E][NC][NPAIR][2], then the constant modes [E][NC]
  for (int j = tid; j < NPAIR * NC * E; j += NT) {
    const int rank = j / (NC * E), ev = j - rank * (NC * E), e = ev / NC;
    int a1, a2;
    pr_by_rank<N>(rank, a1, a2);
    const int pr = pr_of(N, a1, a2), n3 = N - a1 - a2;
    double ent = 0.0, eab = 0.0;
    const double* wt = (ent_mode && e < ne) ? A.wt + ((size_t)e0 * NC + ev) * Np + off_of(N, a1, a2) : nullptr;
    double* cons = (ent_mode && pr == 0) ? pe + E * NC * NPAIR * 2 + ev : nullptr;
    modeB_dispatch<N, true>(n3, S + ev * Z::SEV + pr * N, cons, ent, eab, wt);
    if (ent_mode) {
      pe[(ev * NPAIR + pr) * 2] = ent;
      pe[(ev * NPAIR + pr) * 2 + 1] = eab;
    }
  }
  __syncthreads();
  if (ent_mode) {  // deterministic per-element sums (fixed order)
    for (int e = tid; e < ne; e += NT) {
      double s0 = 0.0, s1 = 0.0;
      for (int q = 0; q < NC * NPAIR; ++q) {
        s0 += pe[(e * NC * NPAIR + q) * 2];
        s1 += pe[(e * NC * NPAIR + q) * 2 + 1];
      }
      double* pp = A.part + (e0 + e) * (2 + NC);
      pp[0] = s0;
      pp[1] = s1;
      for (int v = 0; v < NC; ++v) pp[2 + v] = pe[E * NC * NPAIR * 2 + e * NC + v] / A.c0;
    }
  }
  // ---- A2: V steps 2-3, W / J~, V^T steps 1-2, lane = (e, v, c) (all threads, as A1) ----
  cp_async_wait_all();
  __syncthreads();
  {
    const bool act = tid < NC * E * N;
    const int ev = act ? tid / N : 0, c = act ? tid - ev * N : 0, e = ev / NC;
    modeA_mid<N>(S + ev * Z::SEV + c, U + e * UPE + c, act);
  }
  __syncthreads();
  // ---- B2: V^T step 3 -> du~/dt in U[e][v][k] ----
  for (int j = tid; j < NPAIR * NC * E; j += NT) {
    const int rank = j / (NC * E), ev = j - rank * (NC * E);
    int a1, a2;
    pr_by_rank<N>(rank, a1, a2);
    const int pr = pr_of(N, a1, a2), n3 = N - a1 - a2;
    double d0 = 0.0, d1 = 0.0;
    modeB_dispatch<N, false>(n3, S + ev * Z::SEV + pr * N, U + ev * Np + off_of(N, a1, a2), d0, d1, nullptr);
  }
  __syncthreads();
  // ---- epilogue: output or RK4 stage update (R17), coalesced over the CTA's element block ----
  const size_t base = (size_t)e0 * UPE;
  const int nv = ne * UPE;
  const double dt = A.dt;
  for (int k = tid; k < nv; k += NT) {
    const double du = U[k];
    const size_t g = base + k;
    switch (A.mode) {
      case 0:
      case 5:
        A.out[g] = du;
        break;
      case 1:
        A.acc[g] = A.u0[g] + (dt / 6.0) * du;
        A.ustage[g] = A.u0[g] + (0.5 * dt) * du;
        break;
      case 2:
        A.acc[g] += (dt / 3.0) * du;
        A.ustage[g] = A.u0[g] + (0.5 * dt) * du;
        break;
      case 3:
        A.acc[g] += (dt / 3.0) * du;
        A.ustage[g] = A.u0[g] + dt * du;
        break;
      case 4:
        A.out[g] = A.acc[g] + (dt / 6.0) * du;
        break;
    }
  }
}

// W / J~ from geo_vol rows (node order a + N b + N^2 c) into [e][b][a][c]
template <int N>
__global__ void wjinv_permute_kernel(const double* geo_vol, int gvs, int row, int64_t n, double* out) {
  constexpr int Nq = N * N * N;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * Nq) return;
  const int64_t e = t / Nq;
  const int q = (int)(t - e * Nq), b = q / (N * N), a = (q / N) % N, c = q % N;
  out[t] = geo_vol[(size_t)e * gvs + (size_t)row * Nq + a + N * b + N * N * c];
}

}  // namespace esb
