// rhs2.cuh -- K2 (v5): persistent warp-synchronous line-wise flux differencing (product code).
//
// Each warp owns whole eta_k lines ("line groups" of N lanes, floor(32/N) lines per warp).  For one
// direction k a lane keeps its node's entropy-projected state and metric rows in registers, pairs
// with the node (pos+s) mod N of its line for s = 1..floor(N/2) (every unordered pair exactly once,
// P:572), subtracts F from its own accumulator and receives the partner's +F by a warp shuffle.
// The facet-correction pairs whose extrapolation runs along the same lines are done in
// the same pass; their facet-side sums C^T 1 go through a per-warp shared-memory scratch and are
// summed in a fixed order (deterministic, no atomics).  One persistent CTA per SM loops over
// elements; the element's states, metric terms, traces, facet normals, interface fluxes and W/J~
// arrive by bulk asynchronous copies (cp.async.bulk, TMA engine) on two mbarriers, issued for the
// next element as soon as the current one is done with each buffer, so the copies overlap compute.
// The facet correction is subtracted in place from the interface fluxes (computed beforehand by
// iface_kernel), then lifting and the weight-adjusted inverse (in-place transforms) follow.
#pragma once
#include <type_traits>

#include "kernels.cuh"

namespace esb {

// the dynamic shared memory of the flux kernel, visible to its non-inlined helpers so that their
// accesses compile to shared-memory loads and stores
extern __shared__ __align__(16) double smk2[];

// volume-job partner data by shuffle from the partner lane (1), or from shared memory (0); the default
// (-1) shuffles for tetrahedra up to N = 7 (C4, N = 5: flux kernel 0.65 -> 0.63 ms) and loads at N = 9
// (C5: 36.14 ms with loads, 36.38 with shuffles -- more spills at 128 registers)
#ifndef ES_K2_SHFL
#define ES_K2_SHFL -1
#endif
template <int DIM, int N>
__host__ __device__ constexpr bool k2_shfl() {
  return ES_K2_SHFL == 1 || (ES_K2_SHFL == -1 && DIM == 3 && N <= 7);
}
#ifndef ES_K2_NWMAX
#define ES_K2_NWMAX 16  // warps per flux-kernel CTA (4 per SM sub-partition at <= 128 registers)
#endif
// tetrahedra at N = 9 (C5): 12 warps at 168 registers (35.56 ms per RHS) beat 16 at 128 (36.14 ms) once
// the shared-memory bank conflicts were removed (tools/gpu_k2sweep.sh; 14 warps: 47.0 ms)
#ifndef ES_K2_NW9
#define ES_K2_NW9 12
#endif
template <int DIM, int N>
struct Lw {  // line-group layout
  using S = Sz<DIM, N>;
  static constexpr int LPW = 32 / N;                         // lines per warp slot
  static constexpr int NL = DIM == 2 ? N : N * N;            // lines per direction
  static constexpr int SLOTS = (NL + LPW - 1) / LPW;         // warp slots per direction
  static constexpr int NWM = (DIM == 3 && N == 9) ? ES_K2_NW9 : ES_K2_NWMAX;
  static constexpr int NW = SLOTS <= NWM ? SLOTS : NWM;
  static constexpr int NT = NW * 32;
  static constexpr int NS = N / 2;                            // shifts
#ifndef ES_K2_VB
#define ES_K2_VB 2
#endif
  static constexpr int VB = ES_K2_VB;  // volume pair jobs per flux batch (ILP vs registers: 4 spills at N = 9)
};

__host__ __device__ constexpr int ev2(int x) { return (x + 1) & ~1; }

template <int DIM, int N>
struct Rhs2Smem {
  using S = Sz<DIM, N>;
  using W = Lw<DIM, N>;
  // per-CTA constants (staged once by the persistent CTA)
  static constexpr int TB = 5 * N * N + 6 * N + N * N + S::NF;  // line operators, weights, extrapolation, B
  // PKD sum-factorisation tables: 2D only (3D hands the nodal residual to the batched K3, xform3.cuh)
  static constexpr int PS = DIM == 2 ? psi_smem_doubles<DIM, N>() : 0;
  // per element
  static constexpr int PR = S::PRS;                  // rho, v, p, beta, flag (bulk copy of prim)
  static constexpr int GG = ev2(S::NG * S::Nq);      // G_lm              (bulk copy)
  static constexpr int RR = ev2(S::NC * S::Nq);      // nodal residual r; first transform buffer
  static constexpr int PT = DIM == 3 ? S::NC * N * N * N : 0;  // facet-4 partial sums [v][j][a][c]
  static constexpr int UM = DIM == 2 ? ev2(S::NC * S::Np) : S::NC * N * N;  // 2D modal result / 3D facet-4 lift
  static constexpr int FP = S::Nf * S::NC * S::Nqf;  // facet states [z][rho, v, p][f] (bulk copy)
  static constexpr int FB = ev2(S::NF);              // facet beta = rho / p
  static constexpr int FJ = S::Nf * DIM * S::Nqf;    // J n at facet nodes [z][m][f] (bulk copy)
  static constexpr int FS = S::Nf * S::NC * S::Nqf;  // B J_f f* (computed in the prologue), then s = B J_f f* - C^T 1
  static constexpr int FN = S::Nf * S::NC * S::Nqf;  // neighbour traces at this element's facet nodes (cp.async)
  // per-warp reduction scratch of the line sums: SCV variables per round, sized to fit the region
  // it shares with the modal result (all NC at once when there is room)
  // (all NC variables per round: the facet-side line sums are a latency chain per round, and in 3D
  // the region no longer holds the modal result, so it is sized for the scratch)
  // row stride RS of the scratch (>= 32): the line sums read N consecutive doubles of row u at
  // u RS + gq N; RS is chosen so that the LPW x SCV reading lanes fall into distinct shared-memory banks
  // (bank model of tools/banksim.py: 9 instead of 45 wavefronts per round at N = 9)
  static constexpr int RS = N == 9 ? 37 : (N == 3 ? 39 : 33);
  static constexpr int SCV_FIT = W::NW * S::NC * RS <= UM ? S::NC : (UM / (W::NW * RS) >= 1 ? UM / (W::NW * RS) : 1);
  static constexpr int SCV = DIM == 3 ? S::NC : SCV_FIT;
  static constexpr int SC = W::NW * SCV * RS;
  static constexpr int WJ0 = ((S::NG * S::Nq) % 2 == 0) ? S::NG * S::Nq : (S::NG + 1) * S::Nq;  // first even row
  static constexpr int WJN = ((S::NG * S::Nq) % 2 == 0) ? 2 * S::Nq : ev2(S::Nq);                // doubles copied
  static constexpr int WJOFF = ((S::NG * S::Nq) % 2 == 0) ? S::Nq : 0;  // W / J~ within the copied rows
  static constexpr int PB = PT > RR ? PT : RR;  // facet-4 partials, then the second transform buffer
  static constexpr int SCU = SC > UM ? SC : UM;   // warp scratch, then modal result + facet-4 lifting
  static constexpr int o_tb = 0, o_ps = ev2(o_tb + TB), o_pr = ev2(o_ps + PS), o_g = o_pr + PR, o_r = ev2(o_g + GG),
                       o_pt = ev2(o_r + RR), o_fp = ev2(o_pt + PB), o_fb = ev2(o_fp + FP),
                       o_fj = ev2(o_fb + FB), o_fs = ev2(o_fj + FJ), o_fn = ev2(o_fs + FS), o_sc = ev2(o_fn + FN), o_um = o_sc, o_wj = ev2(o_sc + SCU),
                       total = ev2(o_wj + (DIM == 2 ? 2 * ev2(WJN) : 0));  // 2D: W/J~ double-buffered by element parity
  static_assert(S::PRS <= PR, "prim copy");
  static_assert(total * 8 <= 227 * 1024 - 256, "shared memory");
};

template <int DIM, int N>
__host__ __device__ constexpr size_t rhs2_smem_doubles() {
  return Rhs2Smem<DIM, N>::total;
}

// logarithmic mean and its reciprocal (reading R5); one reciprocal each.  In the Taylor
// branch 1/P(f2) is evaluated as 1/(2(1+g)) = (1 - g + g^2 - g^3)/2, truncation g^4 < 2e-18.
__device__ __forceinline__ double ln_mean_v2(double x, double y) {
  double s = x + y;
  double is = __drcp_rn(s);
  double u = (x - y) * is;
  double f2 = u * u;
  if (f2 < 1e-4) {
    double g = f2 * (1.0 / 3.0 + f2 * (1.0 / 5.0 + f2 * (1.0 / 7.0)));
    return s * (0.5 * (1.0 + g * (-1.0 + g * (1.0 - g))));
  }
  return (y - x) / log(y / x);
}
__device__ __forceinline__ double inv_ln_mean_v2(double x, double y) {
  double s = x + y;
  double is = __drcp_rn(s);
  double u = (x - y) * is;
  double f2 = u * u;
  if (f2 < 1e-4) return (2.0 + f2 * (2.0 / 3.0 + f2 * (2.0 / 5.0 + f2 * (2.0 / 7.0)))) * is;
  return log(y / x) / (y - x);
}

// entropy-projected node state: rho, v, p (p / 2 in the flux kernel's rows, see flux_batch), beta
struct NodeState {
  double r, v[3], p, b;
};

// Ranocha EC flux in direction n (R3)
template <int DIM>
__device__ __forceinline__ void ec_flux_v2(const NodeState& A, const NodeState& B, const double* n,
                                           double gm1inv, double* F) {
  double rho_ln = ln_mean_v2(A.r, B.r);
  double ib_ln = inv_ln_mean_v2(A.b, B.b);
  double vn = 0.0, van = 0.0, vbn = 0.0, vdot = 0.0, vav[DIM];
#pragma unroll
  for (int m = 0; m < DIM; ++m) {
    vav[m] = 0.5 * (A.v[m] + B.v[m]);
    vn += vav[m] * n[m];
    van += A.v[m] * n[m];
    vbn += B.v[m] * n[m];
    vdot += A.v[m] * B.v[m];
  }
  double pav = 0.5 * (A.p + B.p);
  double fr = rho_ln * vn;
  F[0] = fr;
#pragma unroll
  for (int m = 0; m < DIM; ++m) F[1 + m] = fr * vav[m] + pav * n[m];
  F[DIM + 1] = fr * (0.5 * vdot + ib_ln * gm1inv) + 0.5 * (A.p * vbn + B.p * van);
}

// warp shuffle of a double as two 32-bit halves (no register moves around inline asm)
__device__ __forceinline__ double shfl_d(double x, int src) {
  int lo = __double2loint(x), hi = __double2hiint(x);
  lo = __shfl_sync(0xffffffffu, lo, src);
  hi = __shfl_sync(0xffffffffu, hi, src);
  return __hiloint2double(hi, lo);
}

// reciprocal: hardware approximation refined by one cubic step r (1 + e + e^2), e = 1 - s r (error
// e^3 ~ 1e-18 from the seed's 9.9e-7; within 1 ulp of the correctly rounded 1/s over 2^26 arguments,
// tools/rcp_check.cu, profiles/r01_v47_rcp_check.json); arguments are positive and normal
__device__ __forceinline__ double rcp_nr(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  const double e = fma(-s, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// one Newton step: relative error ~2^-44 from the ~2^-22 seed.  Used where the reciprocal only
// enters the Taylor argument f2 = ((x-y)/(x+y))^2 of the logarithmic mean, whose contribution
// g = f2/3 + ... < 4e-5 makes that error ~1e-18 in the mean (R5)
__device__ __forceinline__ double rcp_nr1(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  return fma(r, fma(-s, r, 1.0), r);
}

// one pair job: the other state lives in shared memory at base[q * stride + idx] (q = rho, v, p)
// and bb[idx] (beta); n is the direction, already scaled by the operator coefficient (f# is linear
// in n), zero for masked jobs -- which makes F exactly zero
template <int DIM>
struct Job {
  const double* base;
  const double* bb;
  int stride, idx;
  double n[DIM];
};

// B Ranocha fluxes (R3) of `me` with the job states, straight-line in the common case: both
// log means take the Taylor branch; a warp-uniform fallback recomputes the members that need the
// log branch (R5).  F[b][v] = f#(me, other_b, n_b).
// CHK = false: the caller guarantees that every pair of the element takes the Taylor branch of
// both logarithmic means (element-wide bound on the spread of rho and beta), so the branch test
// is dropped -- the arithmetic is identical to the checked path for such pairs.
template <int DIM, int B, bool CHK = true>
__device__ __forceinline__ void flux_batch_o(const NodeState& me, const NodeState* o, const Job<DIM>* jb, double gm1inv,
                                             double (*F)[DIM + 2]);
template <int DIM, int B, bool CHK = true>
__device__ __forceinline__ void flux_batch(const NodeState& me, const Job<DIM>* jb, double gm1inv,
                                           double (*F)[DIM + 2]) {
  NodeState o[B];
#pragma unroll
  for (int t = 0; t < B; ++t) {
    const double* q = jb[t].base + jb[t].idx;
    const int st = jb[t].stride;
    o[t].r = q[0];
#pragma unroll
    for (int m = 0; m < DIM; ++m) o[t].v[m] = q[(1 + m) * st];
    o[t].p = q[(DIM + 1) * st];
    o[t].b = jb[t].bb[jb[t].idx];
  }
  flux_batch_o<DIM, B, CHK>(me, o, jb, gm1inv, F);
}
// the same with the other states already in registers (volume jobs: shuffled from the partner lanes)
template <int DIM, int B, bool CHK>
__device__ __forceinline__ void flux_batch_o(const NodeState& me, const NodeState* o, const Job<DIM>* jb, double gm1inv,
                                             double (*F)[DIM + 2]) {
  double rl[B], ib[B], f2r[B], f2b[B];
  bool need = false;
#pragma unroll
  for (int t = 0; t < B; ++t) {
    const double sr = me.r + o[t].r, isr = rcp_nr1(sr), ur = (me.r - o[t].r) * isr;
    f2r[t] = ur * ur;
    // (x + y) / (2 P(f2)), P = 1 + f2/3 + f2^2/5 + f2^3/7, with 1/P = 1 - f2/3 - 4 f2^2/45
    // - 44 f2^3/945 + O(f2^4) (the O(f2^4) term is below 3e-18 for f2 < 1e-4, R5)
    rl[t] = sr * (0.5 + f2r[t] * (-1.0 / 6.0 + f2r[t] * (-2.0 / 45.0 + f2r[t] * (-22.0 / 945.0))));
    const double sb = me.b + o[t].b, isb = rcp_nr(sb), ub = (me.b - o[t].b) * isb;
    f2b[t] = ub * ub;
    ib[t] = (2.0 + f2b[t] * (2.0 / 3.0 + f2b[t] * (2.0 / 5.0 + f2b[t] * (2.0 / 7.0)))) * isb;
    if constexpr (CHK) need |= (f2r[t] >= 1e-4) | (f2b[t] >= 1e-4);
  }
  if (CHK && __any_sync(0xffffffffu, need)) {
#pragma unroll
    for (int t = 0; t < B; ++t) {
      if (f2r[t] >= 1e-4) rl[t] = (o[t].r - me.r) / log(o[t].r / me.r);
      if (f2b[t] >= 1e-4) ib[t] = log(o[t].b / me.b) / (o[t].b - me.b);
    }
  }
#pragma unroll
  for (int t = 0; t < B; ++t) {
    const double* n = jb[t].n;
    // <v>.n = (v_a.n + v_b.n) / 2; <v_m> f = (v_a,m + v_b,m) f / 2
    double van = 0.0, vbn = 0.0, vdot = 0.0;
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      van += me.v[m] * n[m];
      vbn += o[t].v[m] * n[m];
      vdot += me.v[m] * o[t].v[m];
    }
    // the p fields hold p / 2: <p> = p_a/2 + p_b/2, (p_a v_b.n + p_b v_a.n)/2 below (exact scalings)
    const double pav = me.p + o[t].p;
    const double fr = rl[t] * (0.5 * (van + vbn));
    const double hfr = 0.5 * fr;
    F[t][0] = fr;
#pragma unroll
    for (int m = 0; m < DIM; ++m) F[t][1 + m] = hfr * (me.v[m] + o[t].v[m]) + pav * n[m];
    F[t][DIM + 1] = fr * (0.5 * vdot + ib[t] * gm1inv) + (me.p * vbn + o[t].p * van);
  }
}

// ---- bulk asynchronous copies (TMA engine) global -> shared, completing on an mbarrier ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// mbarriers of the flux kernel: element data for the passes (A) / interface fluxes and W/J~ (B)
__shared__ uint64_t k2_barA;

// entropy variables of a primitive state (App. B, R7): w = ((g - s)/(g - 1) - b|v|^2/2, b v, -b),
// s = ln p - g ln rho, b = rho / p
template <int DIM>
__device__ __forceinline__ void wvars(const NodeState& a, double g, double* w) {
  double v2 = 0.0;
#pragma unroll
  for (int m = 0; m < DIM; ++m) v2 += a.v[m] * a.v[m];
  const double s = log(a.p) - g * log(a.r);
  w[0] = (g - s) / (g - 1.0) - 0.5 * a.b * v2;
#pragma unroll
  for (int m = 0; m < DIM; ++m) w[1 + m] = a.b * a.v[m];
  w[DIM + 1] = -a.b;
}
// D = (du/dw)(u(wbar)) (w+ - w-), wbar the mean of the two sides' entropy variables (reading R27).
// du/dw in primitive form, applied without forming the matrix:
//   D_0   = rho (dw_0 + v.dw_v) + E dw_E
//   D_v   = rho v (dw_0 + v.dw_v) + p dw_v + rho h v dw_E
//   D_E   = E dw_0 + rho h v.dw_v + (rho h^2 - g p^2 / (rho (g - 1))) dw_E,  h = (E + p) / rho
// MAT (reading R28): D = |A_n| (du/dw) [w] at the same state, with the Barth-scaled eigenvectors:
//   |v.n| (du/dw)[w] + sum_{+,-} (|v.n +- a| - |v.n|) rho/(2g) (r_+- . [w]) r_+-,
//   r_+- = (1, v +- a n, h +- a v.n), a^2 = g p / rho; lam is unused then
template <int DIM, bool MAT = false>
__device__ __forceinline__ void entropy_jump(const NodeState& um, const NodeState& up, double g, double* D,
                                             const double* nu = nullptr) {
  double wm[DIM + 2], wp[DIM + 2], wb[DIM + 2], dw[DIM + 2];
  wvars<DIM>(um, g, wm);
  wvars<DIM>(up, g, wp);
#pragma unroll
  for (int k = 0; k < DIM + 2; ++k) {
    wb[k] = 0.5 * (wm[k] + wp[k]);
    dw[k] = wp[k] - wm[k];
  }
  // u(wbar): b = -w_last, v = w_v / b, s = g - (g - 1)(w_0 + b|v|^2/2), rho = (b e^s)^(1/(1-g))
  const double b = -wb[DIM + 1];
  double v[DIM], v2 = 0.0, vdw = 0.0;
#pragma unroll
  for (int m = 0; m < DIM; ++m) {
    v[m] = wb[1 + m] / b;
    v2 += v[m] * v[m];
  }
  const double s = g - (g - 1.0) * (wb[0] + 0.5 * b * v2);
  const double r = exp((s + log(b)) / (1.0 - g)), p = r / b;
  const double E = p / (g - 1.0) + 0.5 * r * v2, rh = E + p;
#pragma unroll
  for (int m = 0; m < DIM; ++m) vdw += v[m] * dw[1 + m];
  const double c0 = r * (dw[0] + vdw);
  D[0] = c0 + E * dw[DIM + 1];
#pragma unroll
  for (int m = 0; m < DIM; ++m) D[1 + m] = v[m] * (c0 + rh * dw[DIM + 1]) + p * dw[1 + m];
  D[DIM + 1] = E * dw[0] + rh * vdw + (rh * rh / r - g * p * p / (r * (g - 1.0))) * dw[DIM + 1];
  if constexpr (MAT) {
    const double a = sqrt(g * p / r), h = rh / r;
    double vn = 0.0, adn = 0.0;
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      vn += v[m] * nu[m];
      adn += nu[m] * dw[1 + m];
    }
    const double avn = fabs(vn);
    // r_+- . [w] = dw_0 + v.dw_v +- a n.dw_v + (h +- a v.n) dw_E
    const double base = dw[0] + vdw + h * dw[DIM + 1], sh = a * (adn + vn * dw[DIM + 1]);
    const double km = (fabs(vn - a) - avn) * r / (2.0 * g) * (base - sh);
    const double kp = (fabs(vn + a) - avn) * r / (2.0 * g) * (base + sh);
    D[0] = avn * D[0] + km + kp;
#pragma unroll
    for (int m = 0; m < DIM; ++m) D[1 + m] = avn * D[1 + m] + km * (v[m] - a * nu[m]) + kp * (v[m] + a * nu[m]);
    D[DIM + 1] = avn * D[DIM + 1] + km * (h - a * vn) + kp * (h + a * vn);
  }
}


// interface flux at one facet node (Davis' wave speed P:839): EC flux in the unit normal
// n = J n / J_f of this side plus the dissipation of mode ES (0 none, 1 LLF, 2 entropy jump R27, 3
// matrix R28); returns B J_f f* in out[v * ostride].  um / up: own and neighbour traces (rho, v, p/2) at
// the node with strides; both sides of a face evaluate it with their own normals (partition-independent)
template <int DIM>
__device__ __forceinline__ void iface_node_flux(int es, const double* tm, int sm_, const double* tp, int sp,
                                                const double* Jn, double Bf, double g, double* out, int ostride) {
  constexpr int NC = DIM + 2;
  const double gm1inv = 1.0 / (g - 1.0);
  NodeState um, up;
  um.r = tm[0];
  up.r = tp[0];
#pragma unroll
  for (int m = 0; m < DIM; ++m) {
    um.v[m] = tm[(1 + m) * sm_];
    up.v[m] = tp[(1 + m) * sp];
  }
  um.p = 2.0 * tm[(DIM + 1) * sm_];  // the trace rows hold p / 2
  up.p = 2.0 * tp[(DIM + 1) * sp];
  um.b = um.r / um.p;
  up.b = up.r / up.p;
  double Jf = 0.0;
#pragma unroll
  for (int m = 0; m < DIM; ++m) Jf += Jn[m] * Jn[m];
  Jf = sqrt(Jf);
  double nu[DIM];
#pragma unroll
  for (int m = 0; m < DIM; ++m) nu[m] = Jn[m] / Jf;
  double F[NC];
  ec_flux_v2<DIM>(um, up, nu, gm1inv, F);
  if (es != 0) {  // dissipation with Davis's wave speed
    double vnm = 0.0, vnp = 0.0;
#pragma unroll
    for (int m = 0; m < DIM; ++m) {
      vnm += um.v[m] * nu[m];
      vnp += up.v[m] * nu[m];
    }
    const double lam = fmax(fabs(vnm), fabs(vnp)) + fmax(sqrt(g * um.p / um.r), sqrt(g * up.p / up.r));
    double D[NC];
    if (es == 1) {  // local Lax-Friedrichs on the conservative jump
      double Um[NC], Up[NC];
      cons_of<DIM>(um.r, um.v, um.p, gm1inv, Um);
      cons_of<DIM>(up.r, up.v, up.p, gm1inv, Up);
#pragma unroll
      for (int v = 0; v < NC; ++v) D[v] = Up[v] - Um[v];
    } else if (es == 2) {  // entropy-jump scalar dissipation (R27): (du/dw)(u(wbar)) [w]
      entropy_jump<DIM>(um, up, g, D);
    } else {  // matrix dissipation (R28): |A_n| (du/dw) [w] at u(wbar), no lambda
      entropy_jump<DIM, true>(um, up, g, D, nu);
    }
    const double sc = es == 3 ? 0.5 : 0.5 * lam;
#pragma unroll
    for (int v = 0; v < NC; ++v) F[v] -= sc * D[v];
  }
  const double bj = Bf * Jf;
#pragma unroll
  for (int v = 0; v < NC; ++v) out[v * ostride] = bj * F[v];
}

// Line orderings of the direction passes.  The LPW line groups of a warp take consecutive line
// indices L; (l0, l1) = (L mod N, L / N) name the two fixed coordinates of the line, swapped where that
// lowers the shared-memory bank conflicts of the warp's LDS.64 of node data (served per half-warp:
// the sixteen 8-byte addresses of a half should fall into distinct 8-byte bank slots mod 16).  Chosen
// per (N, k) with the bank model of tools/banksim.py and confirmed by ncu (excess shared wavefronts
// of the flux kernel 174M -> 91M at N = 9): the eta3 pass swaps (partner loads 4 -> 3 wavefronts per
// instruction at N = 9), the eta2 pass swaps so that the facet-4 partner loads become broadcasts
// across the warp's lines.
__host__ __device__ constexpr bool line_swap(int DIM, int N, int k) {
  return DIM == 3 && ((k == 1 && (N == 5 || N == 6 || N == 7 || N == 9)) || (k == 2 && (N == 7 || N == 9)));
}
template <int DIM, int N, int k>
__device__ __forceinline__ void line_coords(int L, int pos, int& ca, int& cb, int& cc) {
  int l0 = L % N, l1 = L / N;
  if constexpr (line_swap(DIM, N, k)) {
    const int t = l0;
    l0 = l1;
    l1 = t;
  }
  if constexpr (k == 0) {
    ca = pos;
    cb = l0;
    cc = l1;
  } else if constexpr (k == 1) {
    ca = l0;
    cb = pos;
    cc = l1;
  } else {
    ca = l0;
    cb = l1;
    cc = pos;
  }
  if constexpr (DIM == 2) cc = 0;
}

// ---- modal (compressed) metric storage (es_options.metric_storage = 1) ----
// The element's metric arrives as PKD coefficients g~ [NG][Np] (bulk copy into the head of the G
// region) and is expanded here to G = V g~ at the volume nodes -- exact, the metric terms being
// polynomials of degree <= p (R33) -- by the sum-factorised steps of u = V u~:
//   X[v][pr][c] = sum_a3 psi3[s][a3][c] g~[v][off(pr) + a3]                  items (pr, v), pr-major
//   G[v][a + N b + N^2 c] = sum_a1 psi1[a1][a] sum_a2 psi2[a1][a2][b] X[v][pr(a1, a2)][c]   items (b, v, c)
// with the tables from constant memory (this unit's c_psi<N>, uploaded for K1), so the table reads of
// a warp touch at most a few distinct rows.  X is scratch in the residual / facet-4 regions, both free
// before the passes.  The caller's barrier completes the second step.
template <int N>
__device__ __forceinline__ void metric_expand_3d(double* sG, double* X, int tid, int nt) {
  constexpr int NG = 9, NPAIR = N * (N + 1) / 2, Np = N * (N + 1) * (N + 2) / 6, Nq = N * N * N;
  for (int it = tid; it < NPAIR * NG; it += nt) {
    const int pr = it / NG, v = it - pr * NG;
    int a1 = 0, base = 0, off = 0;  // pr -> (a1, a2) and the first mode of the pair (a1-major nested, R9)
    while (pr >= base + (N - a1)) {
      base += N - a1;
      off += (N - a1) * (N - a1 + 1) / 2;
      ++a1;
    }
    const int a2 = pr - base, s = a1 + a2, n3 = N - s;
    off += a2 * (N - a1) - a2 * (a2 - 1) / 2;
    const double* gm = sG + v * Np + off;
    double x[N];
#pragma unroll
    for (int c = 0; c < N; ++c) x[c] = 0.0;
#pragma unroll
    for (int a3 = 0; a3 < N; ++a3)
      if (a3 < n3) {
        const double gv = gm[a3];
#pragma unroll
        for (int c = 0; c < N; ++c) x[c] = fma(c_psi<N>.p3[(s * N + a3) * N + c], gv, x[c]);
      }
    double* xo = X + (v * NPAIR + pr) * N;
#pragma unroll
    for (int c = 0; c < N; ++c) xo[c] = x[c];
  }
  __syncthreads();
  for (int q = tid; q < N * NG * N; q += nt) {
    const int b = q / (NG * N), r = q - b * (NG * N), v = r / N, c = r - v * N;
    double t2[N], y[N];
#pragma unroll
    for (int a1 = 0; a1 < N; ++a1) {
      const int prs = a1 * N - a1 * (a1 - 1) / 2;
      double t = 0.0;
#pragma unroll
      for (int a2 = 0; a2 < N - a1; ++a2) t = fma(c_psi<N>.p2[(a1 * N + a2) * N + b], X[(v * NPAIR + prs + a2) * N + c], t);
      t2[a1] = t;
    }
    psi1_apply_eo<N>(t2, y);
    double* go = sG + v * Nq + N * b + N * N * c;
#pragma unroll
    for (int a = 0; a < N; ++a) go[a] = y[a];
  }
}

template <int DIM, int N>
__device__ __forceinline__ void k2_epilogue_2d(const RhsArgs& A, int64_t e, unsigned it);

// one element of the flux kernel (the body of the persistent loop); MM: modal metric storage
template <int DIM, int N, bool EQ, bool DN = false, bool CNT = false, bool MM = false>
__device__ __forceinline__ void k2_element(const RhsArgs& A, int64_t idx, unsigned it) {
  using S = Sz<DIM, N>;
  using W = Lw<DIM, N>;
  using L = Rhs2Smem<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf, NT = W::NT, NS = W::NS;
  double* sP = smk2 + L::o_pr;  // [DIM+3][Nq]: rho, v_1..v_d, p, beta
  double* sG = smk2 + L::o_g;   // [NG][Nq]: G_lm at (l*DIM+m)
  double* sR = smk2 + L::o_r;   // [NC][Nq] nodal residual
  double* pt = smk2 + L::o_pt;  // [NC][N(j)][N(a)][N(c)] facet-4 partials
  double* sU = smk2 + L::o_um;  // [NC][Np] modal result + [NC][N][N] facet-4 lifting (aliases the scratch)
  double* fP = smk2 + L::o_fp;  // [Nf][NC][Nqf] facet states rho, v, p
  double* fB = smk2 + L::o_fb;  // [Nf*Nqf] facet beta
  double* fJ = smk2 + L::o_fj;  // [Nf][DIM][Nqf] J n
  double* fS = smk2 + L::o_fs;  // [Nf][NC][Nqf] B J_f f*, then s = B J_f f* - C^T 1
  double* tb = smk2 + L::o_tb;
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

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* scr = smk2 + L::o_sc + warp * L::SCV * L::RS;
  const double g = A.gamma, gm1inv = 1.0 / (g - 1.0);
  auto elem_of = [&](int64_t idx) { return A.elem_list ? A.elem_list[idx] : idx; };
  // bulk copies of one element's data (cp.async.bulk, TMA engine) onto the two mbarriers
  auto issue_A = [&](int64_t e, unsigned buf) {
    constexpr unsigned bP = S::PRS * 8, bG = (MM ? ev2(S::NG * Np) : ev2(S::NG * Nq)) * 8, bF = L::FP * 8,
                       bJ = L::FJ * 8, bW = DIM == 2 ? L::WJN * 8 : 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&k2_barA, bP + bG + bF + bJ + bW);
    bulk_g2s(sP, A.prim + (size_t)e * S::PRS, bP, &k2_barA);
    if constexpr (MM)  // modal metric storage: the PKD coefficients g~ [NG][Np] (+ pad), expanded below
      bulk_g2s(sG, A.gmod + (size_t)e * ev2(S::NG * Np), bG, &k2_barA);
    else
      bulk_g2s(sG, A.geo_vol + (size_t)e * S::GVS, bG, &k2_barA);
    bulk_g2s(fP, A.trace + (size_t)e * L::FP, bF, &k2_barA);
    bulk_g2s(fJ, A.geo_face + (size_t)e * L::FJ, bJ, &k2_barA);
    if constexpr (DIM == 2) bulk_g2s(smk2 + L::o_wj + buf * ev2(L::WJN), A.geo_vol + (size_t)e * S::GVS + L::WJ0, bW, &k2_barA);
  };
  // the neighbour traces of an element's facet nodes, gathered by 8-byte asynchronous copies in this
  // element's node order (the face permutation P:736-741 applied by the copy); they land during the
  // previous element's passes
  auto prefetch_nbr = [&](int64_t e) {
    double* fN = smk2 + L::o_fn;
    for (int zf = tid; zf < S::Nf * Nqf; zf += NT) {  // one facet node per item, its NC variables in turn
      const int z = zf / Nqf, f = zf - z * Nqf;
      const int64_t slot = A.face_slot[e * S::Nf + z];
      const int rf = A.face_reflect[e * S::Nf + z];
      const int fo = DIM == 2 ? (rf ? N - 1 - f : f) : (rf ? (N - 1 - f % N) + N * (f / N) : f);
      const double* src = A.trace + (size_t)slot * NC * Nqf + fo;
      double* dst = fN + z * NC * Nqf + f;
#pragma unroll
      for (int v = 0; v < NC; ++v) cp_async8(dst + v * Nqf, src + v * Nqf);
    }
    cp_async_commit();
  };
  const int grp = lane / N, pos = lane - grp * N;
  const bool lane_ok = grp < W::LPW;
  const int64_t e = elem_of(idx);
  const int64_t nidx = idx + gridDim.x;
  const bool has_next = nidx < A.n_elem;
  const double* gv = A.geo_vol + (size_t)e * S::GVS;
  // optional phase clock stamps (diagnostics, ES_PHASE_TIMING)
  auto stamp = [&](int k) {
    #ifdef ES_STAMPS  // diagnostics build only (tools/build.py with ES_STAMPS=1)
    if (A.dbg && tid == 0 && idx < 4096) A.dbg[idx * 16 + k] = clock64();
#else
    (void)k;
#endif
  };
  // flux-evaluation counters of the counting instantiation (CNT): evaluations with a nonzero operator
  // coefficient in the volume (cv) and facet-correction (cf) passes, every evaluation the lane issued,
  // masked or not (ci), and the interface fluxes (cI) -- observed in the kernel, compared with the
  // oracle's counted loops
  int cv = 0, cf = 0, ci = 0, cI = 0;
  stamp(0);
  mbar_wait(&k2_barA, it & 1);
  if constexpr (MM) {  // G = V g~ at the volume nodes (scratch: the residual and facet-4 regions)
    static_assert(S::NG * S::NPAIR * N <= L::o_fp - L::o_r, "metric expansion scratch");
    if constexpr (DIM == 3) {
      metric_expand_3d<N>(sG, sR, tid, NT);
    } else {
      const PsiS T = psi_tables<DIM, N>(smk2 + L::o_ps);
      modal_to_nodal<DIM, N, S::NG>(T, sG, sG, sR, nullptr);
    }
  }
  // facet beta = rho / p = (rho / (p/2)) / 2 (the volume beta rows and the element's all-Taylor flag
  // come from K1; the state rows hold p / 2)
  for (int fz = tid; fz < NF; fz += NT) {
    const double* q = fP + (fz / Nqf) * NC * Nqf + fz % Nqf;
    fB[fz] = 0.5 * (q[0] / q[(DIM + 1) * Nqf]);
  }
  cp_async_wait_all();  // this element's neighbour traces
  __syncthreads();
  // interface fluxes at the element's facet nodes, B J_f f*: computed in place
  // over the neighbour traces in fN by threads [t0, t0 + nth)
  double* fN = smk2 + L::o_fn;
  auto compute_fstar = [&](int t, int nth, double* dst) {
    for (int fz = t; fz < NF; fz += nth) {
      const int z = fz / Nqf, f = fz - z * Nqf;
      double Jn[DIM];
#pragma unroll
      for (int m = 0; m < DIM; ++m) Jn[m] = fJ[(z * DIM + m) * Nqf + f];
      iface_node_flux<DIM>(A.es, fP + z * NC * Nqf + f, Nqf, fN + z * NC * Nqf + f, Nqf, Jn, tB[fz], g,
                           dst + z * NC * Nqf + f, Nqf);
      if constexpr (CNT) ++cI;
    }
  };
  // HIDE (3D line-wise): the warps with one pass-1 slot fewer than the others (27 slots on 16 warps at
  // N = 9) compute the interface fluxes in the slack of pass 1; fS starts from zero, collects -C^T 1
  // in the passes, and f* is added before the lifting.  Otherwise f* goes into fS before the passes.
  constexpr bool HIDE = DIM == 3 && !DN && (W::SLOTS % W::NW != 0) && (W::SLOTS > W::NW);
  if constexpr (HIDE) {
    for (int q = tid; q < S::Nf * NC * Nqf; q += NT) fS[q] = 0.0;
  } else {
    compute_fstar(tid, NT, fS);
  }
  __syncthreads();
  if constexpr (!HIDE)
    if (has_next) prefetch_nbr(elem_of(nidx));  // fN is consumed
  const bool all_taylor = sP[(DIM + 3) * Nq] != 0.0;
  stamp(1);

  auto state_at = [&](int i) {
    NodeState s;
    s.r = sP[i];
#pragma unroll
    for (int m = 0; m < DIM; ++m) s.v[m] = sP[(1 + m) * Nq + i];
    s.p = sP[(DIM + 1) * Nq + i];
    s.b = sP[(DIM + 2) * Nq + i];
    return s;
  };
  auto Gat = [&](int l, int m, int i) { return sG[(l * DIM + m) * Nq + i]; };

  // ---- direction passes, one specialisation per direction k ----
  // DST: 0 = sR = acc (first pass), 1 = sR += acc, 2 = pt = acc (the pt buffer holds a second
  // residual so that two passes can run without a barrier between them); SYNC: end with a barrier
  auto pass = [&](auto kc, auto tc, auto ec, auto dc, auto sc, int woff) {
    constexpr int k = decltype(kc)::value;
    constexpr int DST = decltype(dc)::value;
    constexpr bool SYNC = decltype(sc)::value;
    constexpr bool CHK = !decltype(tc)::value;
    // EQ56: ablation of the paper's per-operator nonzero iteration: one flux per
    // operator S^(l) with a nonzero on this line instead of one flux with the summed normal
    constexpr bool EQ56 = decltype(ec)::value;
    constexpr int NLOP = EQ56 ? (DIM == 3 ? 3 - k : 2 - k) : 1;  // operators evaluated per pair
    constexpr int stride = k == 0 ? 1 : (k == 1 ? N : N * N);
#pragma unroll 1
    // warp w takes the slots s = w - woff (mod NW): the warps with an extra slot rotate between
    // passes that run back to back
    for (int slot = (warp + W::NW - woff) % W::NW; slot < W::SLOTS; slot += W::NW) {
      // the lanes past the last line group (27..31 at N = 9) address the nodes of the last group,
      // which shares their half-warp (same addresses: shared-memory broadcasts, no extra bank
      // wavefronts), with a zero mask
      const int Lidx = slot * W::LPW + (lane_ok ? grp : W::LPW - 1);
      const bool valid = lane_ok && Lidx < W::NL;
      const bool in_range = Lidx < W::NL;
      // node coordinates (a, b, c) and index; line_coords orders the lines of a warp so that its
      // node loads are free of bank conflicts (line_swap)
      int ca, cb, cc;
      line_coords<DIM, N, k>(in_range ? Lidx : 0, pos, ca, cb, cc);
      const int i = in_range ? ca + N * cb + N * N * cc : 0;
      const double vmask = valid ? 1.0 : 0.0;
      NodeState me = state_at(i);
      double gl[3][3];  // own metric rows g^(l)
#pragma unroll
      for (int l = 0; l < DIM; ++l)
#pragma unroll
        for (int m = 0; m < DIM; ++m) gl[l][m] = Gat(l, m, i);
      double acc[NC];
#pragma unroll
      for (int v = 0; v < NC; ++v) acc[v] = 0.0;

      // -- volume pairs on this line: shifts in batches of VB (ILP), exchanged by shuffles --
      // (ES_K2_SHFL: the partner node's state and metric rows come by shuffle from the partner lane,
      // which holds them in registers, instead of from shared memory -- no bank conflicts, and the
      // shared-memory pipe, 56-75 % busy, carries fewer wavefronts)
#pragma unroll
      for (int s0 = 1; s0 <= NS; s0 += W::VB) {
        Job<DIM> jv[W::VB];
        NodeState ov[W::VB];
        double nl[W::VB][NLOP][DIM];  // per-operator normals (summed unless EQ56)
#pragma unroll
        for (int t = 0; t < W::VB; ++t) {
          const int s = s0 + t;
          int pos2 = pos + (s <= NS ? s : 0);
          if (pos2 >= N) pos2 -= N;
          const int j = in_range ? i + (pos2 - pos) * stride : 0;
          const int ix = pos * N + pos2;
          const int gsrc = (lane_ok ? grp : W::LPW - 1) * N + pos2;  // the partner node's lane
          auto Gj = [&](int l, int m) -> double {
            if constexpr (k2_shfl<DIM, N>())
              return shfl_d(gl[l][m], gsrc);
            else
              return Gat(l, m, j);
          };
          if constexpr (k2_shfl<DIM, N>()) {
            ov[t].r = shfl_d(me.r, gsrc);
#pragma unroll
            for (int m = 0; m < DIM; ++m) ov[t].v[m] = shfl_d(me.v[m], gsrc);
            ov[t].p = shfl_d(me.p, gsrc);
            ov[t].b = shfl_d(me.b, gsrc);
          }
          Job<DIM>& jb = jv[t];
          jb.base = sP;
          jb.bb = sP + (DIM + 2) * Nq;
          jb.stride = Nq;
          jb.idx = j;
          const bool half = (N % 2 == 0) && (s == NS);
          const double mk = (s <= NS && !(half && pos >= N / 2)) ? vmask : 0.0;
          if constexpr (CNT) cv += (mk != 0.0) ? NLOP : 0;
          // term l of n_ij = sum_l c A (g_i^(l) + g_j^(l)) goes to slot min(l', NLOP - 1)
          auto put = [&](int slot, int m, double val) {
            if (EQ56)
              nl[t][slot][m] = val;
            else if (slot == 0)
              nl[t][0][m] = val;
            else
              nl[t][0][m] += val;
          };
          if constexpr (DIM == 2) {
            if (k == 0) {
              const double cl = mk * tw[cb], q1 = cl * tQ1[ix], a1 = cl * tA1[ix];
#pragma unroll
              for (int m = 0; m < 2; ++m) {
                put(0, m, q1 * (gl[0][m] + Gj(0, m)));
                put(1, m, a1 * (gl[1][m] + Gj(1, m)));
              }
            } else {
              const double a2 = mk * tw[ca] * tA2[ix];
#pragma unroll
              for (int m = 0; m < 2; ++m) put(0, m, a2 * (gl[1][m] + Gj(1, m)));
            }
          } else {
            if (k == 0) {
              const double cl = mk * 0.5 * tw[cb] * tw3[cc], q1 = cl * tQ1[ix], a1 = cl * tA1[ix];
#pragma unroll
              for (int m = 0; m < 3; ++m) {
                if constexpr (EQ56) {
                  put(0, m, q1 * (gl[0][m] + Gj(0, m)));
                  put(1, m, a1 * (gl[1][m] + Gj(1, m)));
                  put(2, m, a1 * (gl[2][m] + Gj(2, m)));
                } else {  // metric row 1 holds g1 + g2 in this (last) pass
                  put(0, m, q1 * (gl[0][m] + Gj(0, m)) + a1 * (gl[1][m] + Gj(1, m)));
                }
              }
            } else if (k == 1) {
              const double cl = mk * 0.5 * tw[ca] * tw3[cc], a2 = cl * tA2[ix], a3 = cl * tA3[ix];
#pragma unroll
              for (int m = 0; m < 3; ++m) {
                put(0, m, a2 * (gl[1][m] + Gj(1, m)));
                put(1, m, a3 * (gl[2][m] + Gj(2, m)));
              }
            } else {
              const double a4 = mk * 0.125 * tw[ca] * tw[cb] * (1.0 - teta[cb]) * tA4[ix];
#pragma unroll
              for (int m = 0; m < 3; ++m) put(0, m, a4 * (gl[2][m] + Gj(2, m)));
            }
          }
        }
        double Fs[W::VB][NC];
#pragma unroll
        for (int op = 0; op < NLOP; ++op) {
#pragma unroll
          for (int t = 0; t < W::VB; ++t)
#pragma unroll
            for (int m = 0; m < DIM; ++m) jv[t].n[m] = nl[t][op][m];
          double Fo[W::VB][NC];
          if constexpr (k2_shfl<DIM, N>())
            flux_batch_o<DIM, W::VB, CHK>(me, ov, jv, gm1inv, Fo);
          else
            flux_batch<DIM, W::VB, CHK>(me, jv, gm1inv, Fo);
          if constexpr (CNT) ci += W::VB;
#pragma unroll
          for (int t = 0; t < W::VB; ++t)
#pragma unroll
            for (int v = 0; v < NC; ++v) Fs[t][v] = op == 0 ? Fo[t][v] : Fs[t][v] + Fo[t][v];
        }
#pragma unroll
        for (int t = 0; t < W::VB; ++t) {
          const int s = s0 + t;
          if (s > NS) break;
          int pos0 = pos - s;
          if (pos0 < 0) pos0 += N;
          const int src = grp * N + pos0;
#pragma unroll
          for (int v = 0; v < NC; ++v) acc[v] += shfl_d(Fs[t][v], src) - Fs[t][v];  // masked jobs send 0
        }
      }

      // -- facet-correction pairs along the same lines --
      // a facet job: state of facet node (z, f), normal coef (G_i^T nhat + J n_f)/2 with coefficient
      // coef = (R^T B)_if
      auto fjob_h = [&](Job<DIM>& jb, int z, int f, double c2, const double* gtn) {  // c2 = coef / 2, masked
        jb.base = fP + z * NC * Nqf;
        jb.bb = fB + z * Nqf;
        jb.stride = Nqf;
        jb.idx = f;
#pragma unroll
        for (int m = 0; m < DIM; ++m) jb.n[m] = c2 * (gtn[m] + fJ[(z * DIM + m) * Nqf + f]);
      };
      auto fjob = [&](Job<DIM>& jb, int z, int f, double coef, const double* gtn) {
        fjob_h(jb, z, f, 0.5 * coef * vmask, gtn);
      };
      // facet-side sums over each line group through the warp scratch, in lane order; dest(line, v)
      // returns where the sum of line `gq` goes (nullptr: discard)
      auto line_sums = [&](const double* Fc, auto dest) {
        constexpr int SCV = L::SCV;
#pragma unroll
        for (int v = 0; v < NC; ++v) acc[v] -= Fc[v];
#pragma unroll
        for (int v0 = 0; v0 < NC; v0 += SCV) {
#pragma unroll
          for (int u = 0; u < SCV; ++u)
            if (v0 + u < NC) scr[u * L::RS + lane] = Fc[v0 + u];
          __syncwarp();
          for (int sidx = lane; sidx < W::LPW * SCV; sidx += 32) {
            const int gq = sidx / SCV, u = sidx - gq * SCV, v = v0 + u;
            const double* src = scr + u * L::RS + gq * N;
            double tv[N];  // pairwise tree sum, depth ceil(log2 N)
#pragma unroll
            for (int a = 0; a < N; ++a) tv[a] = src[a];
#pragma unroll
            for (int w = 1; w < N; w *= 2)
#pragma unroll
              for (int a = 0; a + w < N; a += 2 * w) tv[a] += tv[a + w];
            const double sum = tv[0];
            const int Lq = slot * W::LPW + gq;
            if (Lq < W::NL && v < NC) {
              double* d = dest(Lq, v);
              if (d) *d -= sum;  // s = B J_f f* - C^T 1
            }
          }
          __syncwarp();
        }
      };
      if constexpr (DIM == 2) {
        Job<DIM> jf[2];
        if (k == 0) {  // eta1 = +1 (facet 2) and eta1 = -1 (facet 3): facet node b
          const double r2 = 0.70710678118654752440;
          double gtn[2] = {(gl[0][0] + gl[1][0]) * r2, (gl[0][1] + gl[1][1]) * r2};
          double gtn3[2] = {-gl[0][0], -gl[0][1]};
          fjob(jf[0], 1, cb, tlR[ca] * tB[1 * Nqf + cb], gtn);
          fjob(jf[1], 2, cb, tlL[ca] * tB[2 * Nqf + cb], gtn3);
          double Fc[2][NC];
          flux_batch<DIM, 2, CHK>(me, jf, gm1inv, Fc);
          if constexpr (CNT) {
            ci += 2;
            cf += valid ? 2 : 0;
          }
          line_sums(Fc[0], [&](int Lq, int v) { return fS + (1 * NC + v) * Nqf + Lq; });
          line_sums(Fc[1], [&](int Lq, int v) { return fS + (2 * NC + v) * Nqf + Lq; });
        } else {  // eta2 = -1 (facet 1): facet node a
          double gtn[2] = {-gl[1][0], -gl[1][1]};
          fjob(jf[0], 0, ca, tlL[cb] * tB[0 * Nqf + ca], gtn);
          double Fc[1][NC];
          flux_batch<DIM, 1, CHK>(me, jf, gm1inv, Fc);
          if constexpr (CNT) {
            ci += 1;
            cf += valid ? 1 : 0;
          }
          line_sums(Fc[0], [&](int Lq, int v) { return fS + (0 * NC + v) * Nqf + Lq; });
        }
      } else {
        if (k == 0) {  // facets 2 and 3 (eta1 = +1 / -1): facet node (b, c) = line index
          const double r3 = 0.57735026918962576451;
          const int f = cb + N * cc;
          double gtn[3], gtn3[3];
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            gtn[m] = (EQ56 ? gl[0][m] + gl[1][m] + gl[2][m] : gl[0][m] + gl[1][m]) * r3;  // row 1 = g1 + g2 unless EQ56
            gtn3[m] = -gl[0][m];
          }
          Job<DIM> jf[2];
          fjob(jf[0], 1, f, tlR[ca] * tB[1 * Nqf + f], gtn);
          fjob(jf[1], 2, f, tlL[ca] * tB[2 * Nqf + f], gtn3);
          double Fc[2][NC];
          flux_batch<DIM, 2, CHK>(me, jf, gm1inv, Fc);
          if constexpr (CNT) {
            ci += 2;
            cf += valid ? 2 : 0;
          }
          line_sums(Fc[0], [&](int Lq, int v) { return fS + (1 * NC + v) * Nqf + Lq; });
          line_sums(Fc[1], [&](int Lq, int v) { return fS + (2 * NC + v) * Nqf + Lq; });
        } else if (k == 1) {  // facet 1 (eta2 = -1): node (a, c) = line; facet 4 (eta3 = -1): nodes (a, j)
          const int f = ca + N * cc;
          double gtn[3] = {-gl[1][0], -gl[1][1], -gl[1][2]};
          double gt4[3] = {-gl[2][0], -gl[2][1], -gl[2][2]};
          {  // facet 1: one job per lane, summed over the line
            Job<DIM> j1[1];
            fjob(j1[0], 0, f, tlL[cb] * tB[0 * Nqf + f], gtn);
            double F1[1][NC];
            flux_batch<DIM, 1, CHK>(me, j1, gm1inv, F1);
            if constexpr (CNT) {
              ci += 1;
              cf += valid ? 1 : 0;
            }
            line_sums(F1[0], [&](int Lq, int v) {  // facet node (a, c) of line Lq
              int qa, qb, qc;
              line_coords<DIM, N, 1>(Lq, 0, qa, qb, qc);
              return fS + (0 * NC + v) * Nqf + qa + N * qc;
            });
          }
          // facet 4, rotating schedule: at step t lane pos pairs its node (a, b = pos, c) with the
          // facet node (a, j = (pos + t) mod N); the facet-side value travels by shuffle to lane j,
          // which accumulates the sum over b of its facet node (no reduction tree, no scratch)
          double facc[NC];
#pragma unroll
          for (int v = 0; v < NC; ++v) facc[v] = 0.0;
          const double h3 = 0.5 * tl3[cc] * vmask;  // job-independent part of (R^T B)_if / 2
          // B consecutive steps t0 .. t0 + B - 1 in one flux batch
          auto f4batch = [&](auto bc, int t0) {
            constexpr int B = decltype(bc)::value;
            Job<DIM> jq[B];
#pragma unroll
            for (int tt = 0; tt < B; ++tt) {
              int jf = pos + t0 + tt;
              if (jf >= N) jf -= N;
              const int f4 = ca + N * jf;
              fjob_h(jq[tt], 3, f4, (h3 * tli4[jf * N + cb]) * tB[3 * Nqf + f4], gt4);
            }
            double Fb[B][NC];
            flux_batch<DIM, B, CHK>(me, jq, gm1inv, Fb);
            if constexpr (CNT) {
              ci += B;
              cf += valid ? B : 0;
            }
#pragma unroll
            for (int tt = 0; tt < B; ++tt) {
              int p0 = pos - (t0 + tt);
              if (p0 < 0) p0 += N;
              const int src = grp * N + p0;
#pragma unroll
              for (int v = 0; v < NC; ++v) {
                acc[v] -= Fb[tt][v];
                facc[v] += shfl_d(Fb[tt][v], src);
              }
            }
          };
#pragma unroll 1
          for (int t0 = 0; t0 + 1 < N; t0 += 2) f4batch(std::integral_constant<int, 2>{}, t0);
          if constexpr (N % 2 == 1) f4batch(std::integral_constant<int, 1>{}, N - 1);  // no masked job
          if (valid)  // partial over b of facet node (a, j = pos) on line c
#pragma unroll
            for (int v = 0; v < NC; ++v) pt[((v * N + pos) * N + ca) * N + cc] = facc[v];
        }
      }
      // -- residual of this pass (exclusive owner of node i within the pass) --
      if (valid) {
#pragma unroll
        for (int v = 0; v < NC; ++v) {
          if constexpr (DST == 0)
            sR[v * Nq + i] = acc[v];
          else if constexpr (DST == 1)
            sR[v * Nq + i] += acc[v];
          else
            pt[v * Nq + i] = acc[v];
        }
      }
    }
    if constexpr (SYNC) {
      __syncthreads();
      stamp(2 + k);
    }
  };
  using I0 = std::integral_constant<int, 0>;
  using I1 = std::integral_constant<int, 1>;
  using I2 = std::integral_constant<int, 2>;
  using Yes = std::true_type;
  using No = std::false_type;
  // 3D: pass 1 (eta2 lines, with the facet-1 and facet-4 corrections); then the facet-4 sums over
  // c, and g1 + g2 summed in place (the eta1 pass only needs g0 and g1 + g2); then passes 2 and 0
  // back to back without a barrier -- pass 2 accumulates into the freed facet-4 buffer -- and the
  // two residuals are added
  auto passes = [&](auto tc, auto ec) {
    if constexpr (DIM == 3) {
      if constexpr (HIDE) {
        pass(I1{}, tc, ec, I0{}, No{}, 0);
        constexpr int extra = W::SLOTS % W::NW;  // warps below carry one pass-1 slot more
        if (warp >= extra) compute_fstar(tid - extra * 32, (W::NW - extra) * 32, fN);
        __syncthreads();
        stamp(3);
      } else {
        pass(I1{}, tc, ec, I0{}, Yes{}, 0);
      }
      for (int q = tid; q < NC * N * N; q += NT) {  // facet 4: C^T 1 at (a, j) = sum over c of partials
        const int v = q / (N * N), jf = (q / N) % N, a = q % N;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) s += pt[((v * N + jf) * N + a) * N + c];
        fS[(3 * NC + v) * Nqf + a + N * jf] -= s;
      }
      if constexpr (!decltype(ec)::value)
        for (int q = tid; q < DIM * Nq; q += NT) sG[DIM * Nq + q] += sG[2 * DIM * Nq + q];
      __syncthreads();
      pass(I2{}, tc, ec, I2{}, No{}, 0);
      pass(I0{}, tc, ec, I1{}, Yes{}, W::SLOTS % W::NW);
      for (int q = tid; q < NC * Nq; q += NT) sR[q] += pt[q];
      if constexpr (HIDE)  // s = B J_f f* - C^T 1
        for (int q = tid; q < S::Nf * NC * Nqf; q += NT) fS[q] += fN[q];
      __syncthreads();
      if constexpr (HIDE)
        if (has_next) prefetch_nbr(elem_of(nidx));  // fN is consumed
    } else {
      pass(I0{}, tc, ec, I0{}, Yes{}, 0);
      pass(I1{}, tc, ec, I1{}, Yes{}, 0);
    }
  };
  // brute-force ablation (volume_mode 2): every ordered pair (i, j) of volume
  // nodes with the dense S^(l) (zeros included) and every (node, facet node) pair with the dense
  // R^T B; node i owns r_i = -sum_j f#(u_i, u_j, n_ij) - sum_(z,f) f#(u_i, u_f, n_if) (each pair is
  // evaluated from both sides, S skew), facet node f owns s_f -= sum_i f#(u_i, u_f, n_if)
  auto dense_passes = [&]() {
    // all lanes run every iteration (flux_batch takes a warp vote): idle lanes and the i = j pair
    // evaluate with a zero normal, which makes F exactly zero
    const double* Sd = A.sdense;
    const double* RBd = A.rbdense;
    for (int i0 = 0; i0 < Nq; i0 += NT) {
      const int ii = i0 + tid;
      const bool ok = ii < Nq;
      const int i = ok ? ii : 0;
      const NodeState me = state_at(i);
      double gl[3][3], acc[NC];
#pragma unroll
      for (int l = 0; l < DIM; ++l)
#pragma unroll
        for (int m = 0; m < DIM; ++m) gl[l][m] = Gat(l, m, i);
#pragma unroll
      for (int v = 0; v < NC; ++v) acc[v] = 0.0;
      for (int j = 0; j < Nq; ++j) {
        const bool use = ok && j != i;
        Job<DIM> jb[1];
        jb[0].base = sP;
        jb[0].bb = sP + (DIM + 2) * Nq;
        jb[0].stride = Nq;
        jb[0].idx = j;
#pragma unroll
        for (int m = 0; m < DIM; ++m) {
          double nm = 0.0;
#pragma unroll
          for (int l = 0; l < DIM; ++l) nm += __ldg(&Sd[((size_t)l * Nq + j) * Nq + i]) * (gl[l][m] + Gat(l, m, j));
          jb[0].n[m] = use ? nm : 0.0;
        }
        double F[1][NC];
        flux_batch<DIM, 1, true>(me, jb, gm1inv, F);
#pragma unroll
        for (int v = 0; v < NC; ++v) acc[v] -= F[0][v];
      }
      for (int fz = 0; fz < NF; ++fz) {
        const int z = fz / Nqf, f = fz - z * Nqf;
        const double c2 = ok ? 0.5 * __ldg(&RBd[(size_t)fz * Nq + i]) : 0.0;
        Job<DIM> jb[1];
        jb[0].base = fP + z * NC * Nqf;
        jb[0].bb = fB + z * Nqf;
        jb[0].stride = Nqf;
        jb[0].idx = f;
#pragma unroll
        for (int m = 0; m < DIM; ++m) {
          double gtn = 0.0;
#pragma unroll
          for (int l = 0; l < DIM; ++l) gtn += A.nhat[z * 3 + l] * gl[l][m];
          jb[0].n[m] = c2 * (gtn + fJ[(z * DIM + m) * Nqf + f]);
        }
        double F[1][NC];
        flux_batch<DIM, 1, true>(me, jb, gm1inv, F);
#pragma unroll
        for (int v = 0; v < NC; ++v) acc[v] -= F[0][v];
      }
      if (ok)
#pragma unroll
        for (int v = 0; v < NC; ++v) sR[v * Nq + i] = acc[v];
    }
    for (int f0 = 0; f0 < NF; f0 += NT) {
      const int fzz = f0 + tid;
      const bool ok = fzz < NF;
      const int fz = ok ? fzz : 0, z = fz / Nqf, f = fz - z * Nqf;
      double sacc[NC];
#pragma unroll
      for (int v = 0; v < NC; ++v) sacc[v] = 0.0;
      for (int i = 0; i < Nq; ++i) {
        const NodeState me = state_at(i);
        const double c2 = ok ? 0.5 * __ldg(&RBd[(size_t)fz * Nq + i]) : 0.0;
        Job<DIM> jb[1];
        jb[0].base = fP + z * NC * Nqf;
        jb[0].bb = fB + z * Nqf;
        jb[0].stride = Nqf;
        jb[0].idx = f;
#pragma unroll
        for (int m = 0; m < DIM; ++m) {
          double gtn = 0.0;
#pragma unroll
          for (int l = 0; l < DIM; ++l) gtn += A.nhat[z * 3 + l] * Gat(l, m, i);
          jb[0].n[m] = c2 * (gtn + fJ[(z * DIM + m) * Nqf + f]);
        }
        double F[1][NC];
        flux_batch<DIM, 1, true>(me, jb, gm1inv, F);
#pragma unroll
        for (int v = 0; v < NC; ++v) sacc[v] += F[0][v];
      }
      if (ok)
#pragma unroll
        for (int v = 0; v < NC; ++v) fS[(z * NC + v) * Nqf + f] -= sacc[v];
    }
    __syncthreads();
  };
  if constexpr (DN) {
    dense_passes();
  } else {
    // the ablation (EQ) is its own kernel instantiation: the production path keeps its registers
    if (all_taylor)  // uniform over the CTA
      passes(std::true_type{}, std::integral_constant<bool, EQ>{});
    else
      passes(std::false_type{}, std::integral_constant<bool, EQ>{});
  }
  if constexpr (CNT) {  // per-element totals: warp sums, one atomic per warp and counter
    cv = __reduce_add_sync(0xffffffffu, cv);
    cf = __reduce_add_sync(0xffffffffu, cf);
    ci = __reduce_add_sync(0xffffffffu, ci);
    cI = __reduce_add_sync(0xffffffffu, cI);
    if (lane == 0) {
      atomicAdd(A.counts + e * 4 + 3, (unsigned long long)cI);
      atomicAdd(A.counts + e * 4 + 0, (unsigned long long)cv);
      atomicAdd(A.counts + e * 4 + 1, (unsigned long long)cf);
      atomicAdd(A.counts + e * 4 + 2, (unsigned long long)ci);
    }
  }
  // states, metrics and facet inputs are dead: the next element's copies land during the epilogue
  if (tid == 0 && has_next) issue_A(elem_of(nidx), (it + 1) & 1);
  stamp(5);
  // ---- lifting r -= R^T s; facet 4 sum-factorised: t4[v][a][b] = sum_j l_b(eta3_j) s4[v][a + N j] ----
  if constexpr (DIM == 3) {
    double* t4 = sU;
    for (int q = tid; q < NC * N * N; q += NT) {
      const int v = q / (N * N), b = (q / N) % N, a = q % N;
      const double* s4 = fS + (3 * NC + v) * Nqf + a;
      double t = 0.0;
#pragma unroll
      for (int jf = 0; jf < N; ++jf) t = fma(tli4[jf * N + b], s4[N * jf], t);
      t4[(v * N + b) * N + a] = t;
    }
    __syncthreads();
  }
  if constexpr (DIM == 3) {
    // nodal residual r = sR - R^T s, written as r[e][v][b][a][c] (c fastest: the layout the batched
    // weight-adjusted inverse K3 reads coalesced, xform3.cuh); K3 applies P:593 and the RK update
    const double* t4 = sU;
    double* rg = A.rbuf + (size_t)e * NC * Nq;
    for (int rq = tid; rq < Nq; rq += NT) {  // one node per item (index decoded once), its NC variables in turn
      const int b = rq / (N * N), a = (rq / N) % N, c = rq % N;
      const int i = a + N * b + N * N * c;
      const double lb = tlL[b], ra = tlR[a], la = tlL[a], l3 = tl3[c];
      const double* f0 = fS + a + N * c;
      const double* f12 = fS + NC * Nqf + b + N * c;
      const double* t4p = t4 + b * N + a;
#pragma unroll
      for (int v = 0; v < NC; ++v) {
        const double t = lb * f0[v * Nqf] + ra * f12[v * Nqf] + la * f12[(NC + v) * Nqf] + l3 * t4p[v * N * N];
        rg[v * Nq + rq] = sR[v * Nq + i] - t;
      }
    }
    __syncthreads();
    stamp(7);
    return;
  } else {
    for (int i = tid; i < Nq; i += NT) {
      const int a = i % N, b = (i / N) % N;
#pragma unroll
      for (int v = 0; v < NC; ++v) {
        const double t = tlL[b] * fS[(0 * NC + v) * Nqf + a] + tlR[a] * fS[(1 * NC + v) * Nqf + b] +
                         tlL[a] * fS[(2 * NC + v) * Nqf + b];
        sR[v * Nq + i] -= t;
      }
    }
    __syncthreads();
    stamp(7);
    k2_epilogue_2d<DIM, N>(A, e, it);
  }
}

// 2D epilogue of the flux kernel: d u~/dt = V^T W/J~ V (V^T r) in place, then the output /
// RK4 stage update / entropy partials (3D runs this in the batched K3, xform3.cuh)
template <int DIM, int N>
__device__ __forceinline__ void k2_epilogue_2d(const RhsArgs& A, int64_t e, unsigned it) {
  using S = Sz<DIM, N>;
  using W = Lw<DIM, N>;
  using L = Rhs2Smem<DIM, N>;
  constexpr int NC = S::NC, Np = S::Np, NT = W::NT;
  double* sR = smk2 + L::o_r;
  double* pt = smk2 + L::o_pt;
  double* sU = smk2 + L::o_um;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto stamp = [&](int k) {
#ifdef ES_STAMPS
    if (A.dbg && tid == 0 && e < 4096) A.dbg[e * 16 + k] = clock64();
#else
    (void)k;
#endif
  };
  const double* sWJ = smk2 + L::o_wj + (it & 1) * ev2(L::WJN) + L::WJOFF;  // [Nq] W / J~

  // ---- d u~/dt = V^T W/J~ V (V^T r), transforms in place in sR ----
  // ping-pong between sR and the dead facet-4 partial buffer pt (both [NC][Nq]); 3D steps may
  // write their second scratch over the already consumed input
  const PsiS T = psi_tables<DIM, N>(smk2 + L::o_ps);
  if constexpr (DIM == 3)
    nodal_to_modal<DIM, N, NC, 2>(T, sR, sU, sR, pt);
  else
    nodal_to_modal<DIM, N, NC>(T, sR, sU, pt, nullptr);
  stamp(8);
  if (A.mode == 5) {  // entropy production sum w~ . (V^T r) and conservation (V^T r)_0 / c0
    double loc = 0.0, la = 0.0;
    for (int k = tid; k < NC * Np; k += NT) {
      double t = A.wt[(size_t)e * NC * Np + k] * sU[k];
      loc += t;
      la += fabs(t);
    }
    for (int o = 16; o > 0; o >>= 1) {
      loc += __shfl_down_sync(0xffffffffu, loc, o);
      la += __shfl_down_sync(0xffffffffu, la, o);
    }
    __shared__ double red[2][W::NW];
    if (lane == 0) {
      red[0][warp] = loc;
      red[1][warp] = la;
    }
    __syncthreads();
    if (tid == 0) {
      double s0 = 0.0, s1 = 0.0;
      for (int wv = 0; wv < W::NW; ++wv) {
        s0 += red[0][wv];
        s1 += red[1][wv];
      }
      double* pe2 = A.part + (size_t)e * (2 + NC);
      pe2[0] = s0;
      pe2[1] = s1;
      for (int v = 0; v < NC; ++v) pe2[2 + v] = sU[v * Np] / A.c0;
    }
    __syncthreads();
  }
  if constexpr (DIM == 3)
    modal_to_nodal<DIM, N, NC, 2>(T, sU, pt, pt, sR);
  else
    modal_to_nodal<DIM, N, NC>(T, sU, pt, sR, nullptr);
  stamp(9);
  if constexpr (DIM == 3)
    nodal_to_modal<DIM, N, NC, 2>(T, pt, sU, pt, sR, sWJ);  // W / J~ fused into the loads
  else
    nodal_to_modal<DIM, N, NC>(T, pt, sU, sR, nullptr, sWJ);
  stamp(10);
  const size_t base = (size_t)e * NC * Np;
  const double dt = A.dt;
  for (int kk = tid; kk < NC * Np; kk += NT) {
    double du = sU[kk];
    switch (A.mode) {
      case 0:
      case 5:
        A.out[base + kk] = du;
        break;
      case 1:  // classical RK4 stage 1 (R17)
        A.acc[base + kk] = A.u0[base + kk] + (dt / 6.0) * du;
        A.ustage[base + kk] = A.u0[base + kk] + (0.5 * dt) * du;
        break;
      case 2:
        A.acc[base + kk] += (dt / 3.0) * du;
        A.ustage[base + kk] = A.u0[base + kk] + (0.5 * dt) * du;
        break;
      case 3:
        A.acc[base + kk] += (dt / 3.0) * du;
        A.ustage[base + kk] = A.u0[base + kk] + dt * du;
        break;
      case 4:
        A.out[base + kk] = A.acc[base + kk] + (dt / 6.0) * du;
        break;
    }
  }
  __syncthreads();  // sU / sR are reused by the next element
  stamp(11);
}

template <int DIM, int N, bool EQ, bool DN = false, bool CNT = false, bool MM = false>
__device__ __forceinline__ void rhs2_body(DevRef R, const RhsArgs& A) {
  pdl_wait();
  PDL_TRIGGER();
  using S = Sz<DIM, N>;
  using W = Lw<DIM, N>;
  using L = Rhs2Smem<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf, NT = W::NT, NS = W::NS;
  double* sP = smk2 + L::o_pr;  // [DIM+3][Nq]: rho, v_1..v_d, p, beta
  double* sG = smk2 + L::o_g;   // [NG][Nq]: G_lm at (l*DIM+m)
  double* sR = smk2 + L::o_r;   // [NC][Nq] nodal residual
  double* pt = smk2 + L::o_pt;  // [NC][N(j)][N(a)][N(c)] facet-4 partials
  double* sU = smk2 + L::o_um;  // [NC][Np] modal result + [NC][N][N] facet-4 lifting (aliases the scratch)
  double* fP = smk2 + L::o_fp;  // [Nf][NC][Nqf] facet states rho, v, p
  double* fB = smk2 + L::o_fb;  // [Nf*Nqf] facet beta
  double* fJ = smk2 + L::o_fj;  // [Nf][DIM][Nqf] J n
  double* fS = smk2 + L::o_fs;  // [Nf][NC][Nqf] B J_f f*, then s = B J_f f* - C^T 1
  double* tb = smk2 + L::o_tb;
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

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* scr = smk2 + L::o_sc + warp * L::SCV * L::RS;
  const double g = A.gamma, gm1inv = 1.0 / (g - 1.0);
  auto elem_of = [&](int64_t idx) { return A.elem_list ? A.elem_list[idx] : idx; };
  // bulk copies of one element's data (cp.async.bulk, TMA engine) onto the two mbarriers
  auto issue_A = [&](int64_t e, unsigned buf) {
    constexpr unsigned bP = S::PRS * 8, bG = (MM ? ev2(S::NG * Np) : ev2(S::NG * Nq)) * 8, bF = L::FP * 8,
                       bJ = L::FJ * 8, bW = DIM == 2 ? L::WJN * 8 : 0;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&k2_barA, bP + bG + bF + bJ + bW);
    bulk_g2s(sP, A.prim + (size_t)e * S::PRS, bP, &k2_barA);
    if constexpr (MM)  // modal metric storage: the PKD coefficients g~ [NG][Np] (+ pad), expanded below
      bulk_g2s(sG, A.gmod + (size_t)e * ev2(S::NG * Np), bG, &k2_barA);
    else
      bulk_g2s(sG, A.geo_vol + (size_t)e * S::GVS, bG, &k2_barA);
    bulk_g2s(fP, A.trace + (size_t)e * L::FP, bF, &k2_barA);
    bulk_g2s(fJ, A.geo_face + (size_t)e * L::FJ, bJ, &k2_barA);
    if constexpr (DIM == 2) bulk_g2s(smk2 + L::o_wj + buf * ev2(L::WJN), A.geo_vol + (size_t)e * S::GVS + L::WJ0, bW, &k2_barA);
  };
  // the neighbour traces of an element's facet nodes, gathered by 8-byte asynchronous copies in this
  // element's node order (the face permutation P:736-741 applied by the copy); they land during the
  // previous element's passes
  auto prefetch_nbr = [&](int64_t e) {
    double* fN = smk2 + L::o_fn;
    for (int zf = tid; zf < S::Nf * Nqf; zf += NT) {  // one facet node per item, its NC variables in turn
      const int z = zf / Nqf, f = zf - z * Nqf;
      const int64_t slot = A.face_slot[e * S::Nf + z];
      const int rf = A.face_reflect[e * S::Nf + z];
      const int fo = DIM == 2 ? (rf ? N - 1 - f : f) : (rf ? (N - 1 - f % N) + N * (f / N) : f);
      const double* src = A.trace + (size_t)slot * NC * Nqf + fo;
      double* dst = fN + z * NC * Nqf + f;
#pragma unroll
      for (int v = 0; v < NC; ++v) cp_async8(dst + v * Nqf, src + v * Nqf);
    }
    cp_async_commit();
  };
  // ---- per-CTA: barriers, first element's copies, constant tables ----
  if (tid == 0) {
    mbar_init(&k2_barA, 1);
    if ((int64_t)blockIdx.x < A.n_elem) issue_A(elem_of(blockIdx.x), 0);
  }
  if ((int64_t)blockIdx.x < A.n_elem) prefetch_nbr(elem_of(blockIdx.x));
  for (int k = tid; k < N * N; k += NT) {
    tQ1[k] = R.skQ1[k];
    tA1[k] = R.skA1[k];
    tA2[k] = R.skA2[k];
    if constexpr (DIM == 3) {
      tA3[k] = R.skA3[k];
      tA4[k] = R.skA4[k];
      tli4[k] = R.lint4[k];
    }
  }
  for (int k = tid; k < N; k += NT) {
    tw[k] = R.w[k];
    tw3[k] = R.w3[k];
    teta[k] = R.eta[k];
    tlL[k] = R.lL[k];
    tlR[k] = R.lR[k];
    if constexpr (DIM == 3) tl3[k] = R.l3L[k];
  }
  for (int k = tid; k < NF; k += NT) tB[k] = R.Bf[k];
  if constexpr (DIM == 2) stage_psi<DIM, N>(R, smk2 + L::o_ps);  // 3D: no PKD tables in this kernel
  __syncthreads();  // mbarriers initialised and tables staged before anyone uses them

#pragma unroll 1
  for (int64_t idx = blockIdx.x, it = 0; idx < A.n_elem; idx += gridDim.x, ++it) k2_element<DIM, N, EQ, DN, CNT, MM>(A, idx, (unsigned)it);
}

// resident CTAs per SM the register budget is sized for: about 18 warps per SM where shared memory
// allows (small-degree elements have few line slots per CTA), one CTA otherwise
template <int DIM, int N>
__host__ __device__ constexpr int k2_min_blocks() {
  constexpr int smem_fit = (227 * 1024) / (int)(rhs2_smem_doubles<DIM, N>() * 8 + 1024);
  constexpr int want = 18 / Lw<DIM, N>::NW;
  constexpr int b = want < smem_fit ? want : smem_fit;
  return b < 1 ? 1 : b;
}

template <int DIM, int N>
__global__ void __launch_bounds__(Lw<DIM, N>::NT, k2_min_blocks<DIM, N>()) rhs2_kernel(DevRef R, const __grid_constant__ RhsArgs A) {
  rhs2_body<DIM, N, false>(R, A);
}
// modal metric storage (es_options.metric_storage = 1): the production kernel reading g~ instead of G
template <int DIM, int N>
__global__ void __launch_bounds__(Lw<DIM, N>::NT, k2_min_blocks<DIM, N>()) rhs2_mm_kernel(DevRef R, const __grid_constant__ RhsArgs A) {
  rhs2_body<DIM, N, false, false, false, true>(R, A);
}
// counting instantiation (es_count_fluxes): the production kernel with per-element flux counters
template <int DIM, int N>
__global__ void __launch_bounds__(Lw<DIM, N>::NT, k2_min_blocks<DIM, N>()) rhs2_count_kernel(DevRef R, const __grid_constant__ RhsArgs A) {
  rhs2_body<DIM, N, false, false, true>(R, A);
}
template <int DIM, int N>
__global__ void __launch_bounds__(Lw<DIM, N>::NT, 1) rhs2_eq56_count_kernel(DevRef R, const __grid_constant__ RhsArgs A) {
  rhs2_body<DIM, N, true, false, true>(R, A);
}
// ablation: the paper's Eq. num_fluxes per-operator fluxes (es_options.volume_mode = 1)
template <int DIM, int N>
__global__ void __launch_bounds__(Lw<DIM, N>::NT, 1) rhs2_eq56_kernel(DevRef R, const __grid_constant__ RhsArgs A) {
  rhs2_body<DIM, N, true>(R, A);
}
// ablation: brute force over all node pairs with the dense operators (es_options.volume_mode = 2)
template <int DIM, int N>
__global__ void __launch_bounds__(Lw<DIM, N>::NT, 1) rhs2_dense_kernel(DevRef R, const __grid_constant__ RhsArgs A) {
  rhs2_body<DIM, N, false, true>(R, A);
}

}  // namespace esb
