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

#include "psi_const.cuh"
#include "fastmath.cuh"

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
  static constexpr int PRS = ((NC + 1) * Nq + 2) & ~1;  // prim element stride: rho, v, p, beta rows + flag
  static constexpr int KPT = (Nq + 383) / 384;
#ifndef ES_K1_NT9  // tuning experiments: threads per CTA of the per-element kernels at 3D N = 9
  static constexpr int NT = ((Nq + KPT - 1) / KPT + 31) / 32 * 32;
#else
  static constexpr int NT = (DIM == 3 && N == 9) ? ES_K1_NT9 : ((Nq + KPT - 1) / KPT + 31) / 32 * 32;
#endif
};

// device copy of the reference tables (pointers into one device allocation)
struct DevRef {
  const double *eta, *w, *eta3, *w3;
  const double *skQ1, *skA1, *skA2, *skA3, *skA4;
  const double *lL, *lR, *l3L, *lint4;
  const double *psi1, *psi2, *psi3;
  const int *pair_a1, *pair_a2, *pair_off, *mode_pr, *mode_last;
  const double *Bf, *nhat, *Wvol;
  const double* psig;  // the psi tables in the padded layout of psi_tables() (global memory)
};

struct ProjArgs {
  int64_t n_elem;
  const int64_t* elem_list;  // optional element subset
  const double* u;           // [nloc][NC][Np] modal stage input
  const double* geo_vol;     // [nloc][GVS]: [NGV][Nq] + pad
  double* prim;              // [nloc][PRS]: [NC+1][Nq] entropy-projected (rho, v, p, beta = rho/p),
                             // then the element's all-Taylor flag (1.0: every pair takes the Taylor
                             // branch of both logarithmic means, see rhs2.cuh) + pad
  double* trace;             // [slots][NC][Nqf] entropy-projected primitive at facet nodes
  double* wt;                // optional [nloc][NC][Np] projected entropy variables w~
  int* bad;                  // admissibility flag
  double gamma;
  long long* dbg;            // optional [4096][16] phase clock stamps (diagnostics)
  int max_ctas;              // number of SMs (the launcher multiplies by resident CTAs per SM)
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
  int es;                     // interface dissipation: 0 none (EC), 1 LLF, 2 entropy jump (R27), 3 matrix (R28)
  int mode;                   // 0 dudt, 1..4 RK stage 0..3, 5 dudt + entropy partials
  double* out;                // dudt [nloc][NC][Np]
  const double* u0;           // RK state
  double* acc;                // RK accumulator
  double* ustage;             // RK stage input (written)
  double dt;
  const double* wt;           // entropy mode: w~
  double* part;               // entropy mode: [nloc][2 + NC]
  double c0;                  // value of the constant PKD mode (1/sqrt|ref|)
  long long* dbg;             // optional [4096][16] phase clock stamps (diagnostics)
  int max_ctas;               // number of SMs (the launcher multiplies by resident CTAs per SM)
  int eq56;                   // 1: per-operator fluxes (Eq. num_fluxes ablation), 0: line-wise
  const double* sdense;       // volume_mode 2: dense S^(l) [l][j][i]
  const double* rbdense;      // volume_mode 2: dense (R^(z)T B) [z][f][i]
  const double* nhat;         // [Nf][3] reference outward normals
  double* rbuf;               // 3D: nodal residual [nloc][NC][N(b)][N(a)][N(c)] for the batched K3
  unsigned long long* counts; // counting launch: [nloc][4] volume / facet-correction / issued flux evaluations
  const double* gmod;         // modal metric storage: [nloc][ev2(NG Np)] PKD coefficients of G (else null)
};


// ------------------------------------------------------------------------------------------------
// physics: the two-point flux and the logarithmic mean live in rhs2.cuh
// ------------------------------------------------------------------------------------------------
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

// psi tables in shared memory with rows padded to an even length NP (16-byte aligned pairs for
// LDS.128): p1 [N][NP], p2 [N][N][NP], p3 [N][N][NP], then the int pair tables; PSPAD trailing
// doubles keep the over-reads of the last output chunk inside the allocation
template <int N>
__host__ __device__ constexpr int psi_np() { return (N + 1) & ~1; }
constexpr int PSPAD = 4 * 12;
template <int DIM, int N>
__host__ __device__ constexpr int psi_smem_doubles() {
  return N * psi_np<N>() + N * N * psi_np<N>() + (DIM == 3 ? N * N * psi_np<N>() : 0) + PSPAD +
         (3 * (DIM == 2 ? N : N * (N + 1) / 2) + 1) / 2 + 1;
}

// the psi tables at `buf` (layout of stage_psi)
template <int DIM, int N>
__device__ __forceinline__ PsiS psi_tables(double* buf) {
  constexpr int NPAIR = DIM == 2 ? N : N * (N + 1) / 2, NP = psi_np<N>();
  double* p1 = buf;
  double* p2 = p1 + N * NP;
  double* p3 = p2 + N * N * NP;
  int* pi = (int*)(p3 + (DIM == 3 ? N * N * NP : 0) + PSPAD);
  return PsiS{p1, p2, p3, pi, pi + NPAIR, pi + 2 * NPAIR};
}

// stage the tables of R into shared memory at `buf` (psi_smem_doubles<DIM,N>() doubles)
template <int DIM, int N>
__device__ PsiS stage_psi(const DevRef& R, double* buf) {
  constexpr int NPAIR = DIM == 2 ? N : N * (N + 1) / 2, NP = psi_np<N>();
  const PsiS T = psi_tables<DIM, N>(buf);
  double* p1 = (double*)T.p1;
  double* p2 = (double*)T.p2;
  double* p3 = (double*)T.p3;
  for (int k = threadIdx.x; k < N * NP; k += blockDim.x) {
    const int r = k / NP, c = k - r * NP;
    p1[k] = c < N ? R.psi1[r * N + c] : 0.0;
  }
  for (int k = threadIdx.x; k < N * N * NP; k += blockDim.x) {
    const int r = k / NP, c = k - r * NP;
    p2[k] = c < N ? R.psi2[r * N + c] : 0.0;
    if constexpr (DIM == 3) p3[k] = c < N ? R.psi3[r * N + c] : 0.0;
  }
  for (int k = threadIdx.x; k < PSPAD; k += blockDim.x) p1[(N + N * N + (DIM == 3 ? N * N : 0)) * NP + k] = 0.0;
  int* pi = (int*)T.pa1;
  for (int k = threadIdx.x; k < NPAIR; k += blockDim.x) {
    pi[k] = R.pair_a1[k];
    pi[NPAIR + k] = R.pair_a2[k];
    pi[2 * NPAIR + k] = R.pair_off[k];
  }
  return T;
}

// outputs per chunk: a divisor of N when there is one (no wasted FMAs), else 4
template <int N>
__host__ __device__ constexpr int fib_oc() { return N % 3 == 0 ? 3 : (N % 4 == 0 ? 4 : (N % 5 == 0 ? 5 : 4)); }

// Two fibers per work item share every psi load (register blocking): y_f[o] = sum_{i < ni} A[i][o]
// (the two fibers of an item are half a step apart, so that consecutive lanes own consecutive
// fibers: odd strides between lanes, no shared-memory bank conflicts)
// x_f[i] for o < no, f = 0, 1, with A[i][o] = ps[i NP + o] (TR = false) or ps[o NP + i] (TR = true);
// psi pairs are read as 16-byte vectors (padded rows).  Inputs beyond ni are not read (the tables
// vanish there).  Optional per-input scales sc0 / sc1 multiply x (the diagonal W/J~ factor fused
// into the load).  Outputs in chunks of OC, each accumulated over all inputs (independent chains).
template <int N, bool TR>
__device__ __forceinline__ void fiber2(const double* ps, int ni, int no, const double* in0,
                                       const double* in1, int sin, const double* sc0, const double* sc1,
                                       double* out0, double* out1, int sout, bool has1) {
  constexpr int NP = psi_np<N>(), OC = fib_oc<N>();
  double x0[N], x1[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    const bool ok = i < ni;
    x0[i] = ok ? in0[i * sin] : 0.0;
    x1[i] = ok ? in1[i * sin] : 0.0;
    if (sc0) {
      x0[i] *= ok ? sc0[i * sin] : 0.0;
      x1[i] *= ok ? sc1[i * sin] : 0.0;
    }
  }
  if constexpr (!TR && OC % 2 == 1) {
    // odd chunk width: all N outputs at once, each table row read as 16-byte pairs (padded rows);
    // every output is an independent chain over the inputs (no = N on this path)
    double a0[N], a1[N];
#pragma unroll
    for (int o = 0; o < N; ++o) a0[o] = a1[o] = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int q2 = 0; q2 < NP / 2; ++q2) {
        const double2 pv = *reinterpret_cast<const double2*>(ps + i * NP + 2 * q2);
        a0[2 * q2] = fma(pv.x, x0[i], a0[2 * q2]);
        a1[2 * q2] = fma(pv.x, x1[i], a1[2 * q2]);
        if (2 * q2 + 1 < N) {
          a0[2 * q2 + 1] = fma(pv.y, x0[i], a0[2 * q2 + 1]);
          a1[2 * q2 + 1] = fma(pv.y, x1[i], a1[2 * q2 + 1]);
        }
      }
#pragma unroll
    for (int o = 0; o < N; ++o) {
      out0[o * sout] = a0[o];
      if (has1) out1[o * sout] = a1[o];
    }
    return;
  }
  // all output chunks in flight (independent chains); for N a multiple of OC ptxas hoists every
  // table load of every chunk (register blow-up), so the chunks stay sequential there
#pragma unroll(N == 8 ? 1 : N)
  for (int o0 = 0; o0 < N; o0 += OC) {
    if (o0 >= no) break;
    double a0[OC], a1[OC];
#pragma unroll
    for (int q = 0; q < OC; ++q) a0[q] = a1[q] = 0.0;
    if constexpr (!TR) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if constexpr (OC % 2 == 0) {
#pragma unroll
          for (int q2 = 0; q2 < OC / 2; ++q2) {
            const double2 pv = *reinterpret_cast<const double2*>(ps + i * NP + o0 + 2 * q2);
            a0[2 * q2] = fma(pv.x, x0[i], a0[2 * q2]);
            a1[2 * q2] = fma(pv.x, x1[i], a1[2 * q2]);
            a0[2 * q2 + 1] = fma(pv.y, x0[i], a0[2 * q2 + 1]);
            a1[2 * q2 + 1] = fma(pv.y, x1[i], a1[2 * q2 + 1]);
          }
        } else {
#pragma unroll
          for (int q = 0; q < OC; ++q) {
            const double pv = ps[i * NP + o0 + q];
            a0[q] = fma(pv, x0[i], a0[q]);
            a1[q] = fma(pv, x1[i], a1[q]);
          }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < OC; ++q) {
        const double* row = ps + (o0 + q) * NP;
#pragma unroll
        for (int i2 = 0; i2 < NP / 2; ++i2) {
          const double2 pv = *reinterpret_cast<const double2*>(row + 2 * i2);
          a0[q] = fma(pv.x, x0[2 * i2], a0[q]);
          a1[q] = fma(pv.x, x1[2 * i2], a1[q]);
          if (2 * i2 + 1 < N) {
            a0[q] = fma(pv.y, x0[2 * i2 + 1], a0[q]);
            a1[q] = fma(pv.y, x1[2 * i2 + 1], a1[q]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < OC; ++q) {
      if (o0 + q >= no) break;
      out0[(o0 + q) * sout] = a0[q];
      if (has1) out1[(o0 + q) * sout] = a1[q];
    }
  }
}

// K fibers per work item (the flattened steps): x_k = in[k][i sin] (* sc[k][i sin]), outputs
// out[k][o sout] for k < nk; same arithmetic as fiber2 (K = 2) with the table loads shared K ways.
// one fibre, the modal side of runtime length m (the psi3 steps): TR = false: y[o] = sum_{i<m} A[i][o] x[i]
// (N outputs); TR = true: y[o] = sum_i A[o][i] x[i] for o < m.  Loop bounds are compile-time N with the
// modal side predicated (the tables vanish beyond m).
template <int N, bool TR>
__device__ __forceinline__ void fiberK_n(const double* ps, int m, const double* in, int sin, double* out, int sout) {
  constexpr int NP = psi_np<N>();
  double x[N];
#pragma unroll
  for (int i = 0; i < N; ++i) x[i] = (TR || i < m) ? in[i * sin] : 0.0;
  if constexpr (!TR) {
    double a[N];
#pragma unroll
    for (int o = 0; o < N; ++o) a[o] = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i >= m) break;
#pragma unroll
      for (int q2 = 0; q2 < NP / 2; ++q2) {
        const double2 pv = *reinterpret_cast<const double2*>(ps + i * NP + 2 * q2);
        a[2 * q2] = fma(pv.x, x[i], a[2 * q2]);
        if (2 * q2 + 1 < N) a[2 * q2 + 1] = fma(pv.y, x[i], a[2 * q2 + 1]);
      }
    }
#pragma unroll
    for (int o = 0; o < N; ++o) out[o * sout] = a[o];
  } else {
#pragma unroll
    for (int o = 0; o < N; ++o) {
      if (o >= m) break;
      const double* row = ps + o * NP;
      double t = 0.0;
#pragma unroll
      for (int i2 = 0; i2 < NP / 2; ++i2) {
        const double2 pv = *reinterpret_cast<const double2*>(row + 2 * i2);
        t = fma(pv.x, x[2 * i2], t);
        if (2 * i2 + 1 < N) t = fma(pv.y, x[2 * i2 + 1], t);
      }
      out[o * sout] = t;
    }
  }
}

template <int N, bool TR, int K>
__device__ __forceinline__ void fiberK(const double* ps, const double* const* in, int sin, const double* const* sc,
                                       double* const* out, int sout, int nk) {
  constexpr int NP = psi_np<N>(), OC = fib_oc<N>();
  double x[K][N];
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      x[k][i] = in[k][i * sin];
      if (sc) x[k][i] *= sc[k][i * sin];
    }
  if constexpr (!TR && OC % 2 == 1) {  // whole rows as 16-byte pairs (see fiber2)
    double a[K][N];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int o = 0; o < N; ++o) a[k][o] = 0.0;
#pragma unroll
    for (int i = 0; i < N; ++i)
#pragma unroll
      for (int q2 = 0; q2 < NP / 2; ++q2) {
        const double2 pv = *reinterpret_cast<const double2*>(ps + i * NP + 2 * q2);
#pragma unroll
        for (int k = 0; k < K; ++k) {
          a[k][2 * q2] = fma(pv.x, x[k][i], a[k][2 * q2]);
          if (2 * q2 + 1 < N) a[k][2 * q2 + 1] = fma(pv.y, x[k][i], a[k][2 * q2 + 1]);
        }
      }
#pragma unroll
    for (int o = 0; o < N; ++o)
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k < nk) out[k][o * sout] = a[k][o];
    return;
  }
#pragma unroll(N == 8 ? 1 : N)
  for (int o0 = 0; o0 < N; o0 += OC) {  // output chunks in flight (see fiber2)
    double a[K][OC];
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
      for (int q = 0; q < OC; ++q) a[k][q] = 0.0;
    if constexpr (!TR) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if constexpr (OC % 2 == 0) {
#pragma unroll
          for (int q2 = 0; q2 < OC / 2; ++q2) {
            const double2 pv = *reinterpret_cast<const double2*>(ps + i * NP + o0 + 2 * q2);
#pragma unroll
            for (int k = 0; k < K; ++k) {
              a[k][2 * q2] = fma(pv.x, x[k][i], a[k][2 * q2]);
              a[k][2 * q2 + 1] = fma(pv.y, x[k][i], a[k][2 * q2 + 1]);
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < OC; ++q) {
            const double pv = ps[i * NP + o0 + q];
#pragma unroll
            for (int k = 0; k < K; ++k) a[k][q] = fma(pv, x[k][i], a[k][q]);
          }
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < OC; ++q) {
        const double* row = ps + (o0 + q) * NP;
#pragma unroll
        for (int i2 = 0; i2 < NP / 2; ++i2) {
          const double2 pv = *reinterpret_cast<const double2*>(row + 2 * i2);
#pragma unroll
          for (int k = 0; k < K; ++k) {
            a[k][q] = fma(pv.x, x[k][2 * i2], a[k][q]);
            if (2 * i2 + 1 < N) a[k][q] = fma(pv.y, x[k][2 * i2 + 1], a[k][q]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < OC; ++q) {
      if (o0 + q >= N) break;
#pragma unroll
      for (int k = 0; k < K; ++k)
        if (k < nk) out[k][(o0 + q) * sout] = a[k][q];
    }
  }
}

// u = V u~ (modal [NV][Np] -> nodal [NV][Nq]); t1, t2 scratch (t1_size, t2_size)
template <int DIM, int N, int NV, int FB = 2>
__device__ void modal_to_nodal(const PsiS& T, const double* um, double* un, double* t1, double* t2) {
  using S = Sz<DIM, N>;
  constexpr int P = N - 1, NPAIR = S::NPAIR, Np = S::Np, Nq = S::Nq, NVP = (NV + 1) / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (DIM == 2) {
    // t1[v][a1][b] = sum_a2 psi2[a1][a2][b] u[v][off(a1)+a2]; items (a1, variable pair)
    for (int it = tid; it < N * NVP; it += nt) {
      const int a1 = it / NVP, v0 = 2 * (it - a1 * NVP), v1 = v0 + 1 < NV ? v0 + 1 : v0;
      fiber2<N, false>(T.p2 + a1 * N * psi_np<N>(), N - a1, N, um + v0 * Np + T.poff[a1], um + v1 * Np + T.poff[a1], 1, nullptr, nullptr,
                t1 + (v0 * N + a1) * N, t1 + (v1 * N + a1) * N, 1, v1 != v0);
    }
    __syncthreads();
    // u[v][a + N b] = sum_a1 psi1[a1][a] t1[v][a1][b]; items pairs of (v, b) fibers
    constexpr int NFB = NV * N;
    for (int it = tid; it < (NFB + 1) / 2; it += nt) {
      const int q0 = it, q1 = it + (NFB + 1) / 2 < NFB ? it + (NFB + 1) / 2 : it;
      const int v0 = q0 / N, b0 = q0 - v0 * N, v1 = q1 / N, b1 = q1 - v1 * N;
      fiber2<N, false>(T.p1, N, N, t1 + v0 * N * N + b0, t1 + v1 * N * N + b1, N, nullptr, nullptr, un + v0 * Nq + N * b0,
                un + v1 * Nq + N * b1, 1, q1 != q0);
    }
    __syncthreads();
  } else {
    // t1[v][pr][c] = sum_a3 psi3[s][a3][c] u[v][off(pr)+a3]; one (pr, v) fibre per item (225 items at
    // N = 9 fit one round of the CTA: half the critical path of paired fibres)
    for (int it = tid; it < NPAIR * NV; it += nt) {
      const int pr = it / NV, v = it - pr * NV;
      const int sdeg = T.pa1[pr] + T.pa2[pr];
      const double* in[1] = {um + v * Np + T.poff[pr]};
      double* out[1] = {t1 + (v * NPAIR + pr) * N};
      fiberK_n<N, false>(T.p3 + sdeg * N * psi_np<N>(), N - sdeg, in[0], 1, out[0], 1);
    }
    __syncthreads();
    // t2[v][a1][c][b] = sum_a2 psi2[a1][a2][b] t1[v][pr(a1,a2)][c]: one item = the (v, c) fibres of the
    // rows a1 = k and N - 1 - k, N + 1 modal inputs per item whatever k (balanced: a fibre pair of one
    // row a1 = 0 would take 2N); lanes of a warp share k, so the table reads are broadcasts
    constexpr int NFC = NV * N, NK = (N + 1) / 2;
    for (int it = tid; it < NK * NFC; it += nt) {
      const int k = it / NFC, w = it - k * NFC, v = w / N, c = w - v * N;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a1 = h == 0 ? k : N - 1 - k;
        if (h == 1 && a1 == k) break;
        const int prs = a1 * N - a1 * (a1 - 1) / 2;
        fiberK_n<N, false>(T.p2 + a1 * N * psi_np<N>(), N - a1, t1 + (v * NPAIR + prs) * N + c, N,
                           t2 + ((v * N + a1) * N + c) * N, 1);
      }
    }
    __syncthreads();
    // u[v][a + N bc] = sum_a1 psi1[a1][a] t2[v][a1][bc]: one (v, bc) fibre per item, the psi1 table
    // from constant memory (uniform operands) in the even-odd form (psi_const.cuh)
    for (int q = tid; q < NV * N * N; q += nt) {
      const int v = q / (N * N), bc = q - v * N * N;
      const double* in = t2 + v * Nq + bc;
      double x[N], o[N];
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) x[a1] = in[a1 * N * N];
      psi1_apply_eo<N>(x, o);
      double* out = un + v * Nq + N * bc;
#pragma unroll
      for (int a = 0; a < N; ++a) out[a] = o[a];
    }
    __syncthreads();
  }
  (void)P;
}

// u~ = V^T (scale o y) (nodal [NV][Nq] -> modal [NV][Np]); scale: optional per-node factor [Nq]
template <int DIM, int N, int NV, int FB = 2>
__device__ void nodal_to_modal(const PsiS& T, const double* y, double* um, double* t1, double* t2,
                               const double* scale = nullptr) {
  using S = Sz<DIM, N>;
  constexpr int P = N - 1, NPAIR = S::NPAIR, Np = S::Np, Nq = S::Nq, NVP = (NV + 1) / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  if constexpr (DIM == 2) {
    // s1[v][a1][b] = sum_a psi1[a1][a] y[v][a + N b]; items pairs of (v, b) fibers
    constexpr int NFB = NV * N;
    for (int it = tid; it < (NFB + 1) / 2; it += nt) {
      const int q0 = it, q1 = it + (NFB + 1) / 2 < NFB ? it + (NFB + 1) / 2 : it;
      const int v0 = q0 / N, b0 = q0 - v0 * N, v1 = q1 / N, b1 = q1 - v1 * N;
      fiber2<N, true>(T.p1, N, N, y + v0 * Nq + N * b0, y + v1 * Nq + N * b1, 1, scale ? scale + N * b0 : nullptr,
                scale ? scale + N * b1 : nullptr, t1 + v0 * N * N + b0, t1 + v1 * N * N + b1, N, q1 != q0);
    }
    __syncthreads();
    // u[v][off(a1)+a2] = sum_b psi2[a1][a2][b] s1[v][a1][b]; items (a1, variable pair)
    for (int it = tid; it < N * NVP; it += nt) {
      const int a1 = it / NVP, v0 = 2 * (it - a1 * NVP), v1 = v0 + 1 < NV ? v0 + 1 : v0;
      fiber2<N, true>(T.p2 + a1 * N * psi_np<N>(), N, N - a1, t1 + (v0 * N + a1) * N, t1 + (v1 * N + a1) * N, 1, nullptr,
                nullptr, um + v0 * Np + T.poff[a1], um + v1 * Np + T.poff[a1], 1, v1 != v0);
    }
    __syncthreads();
  } else {
    // s2[v][a1][bc] = sum_a psi1[a1][a] y[v][a + N bc] (optional per-node scale): one (v, bc) fibre per
    // item, constant-memory psi1 in the even-odd form (psi_const.cuh)
    for (int q = tid; q < NV * N * N; q += nt) {
      const int v = q / (N * N), bc = q - v * N * N;
      const double* in = y + v * Nq + N * bc;
      double x[N], o[N];
#pragma unroll
      for (int a = 0; a < N; ++a) x[a] = in[a] * (scale ? scale[N * bc + a] : 1.0);
      psi1T_apply_eo<N>(x, o);
      double* out = t2 + v * Nq + bc;
#pragma unroll
      for (int a1 = 0; a1 < N; ++a1) out[a1 * N * N] = o[a1];
    }
    __syncthreads();
    // s1[v][pr(a1,a2)][c] = sum_b psi2[a1][a2][b] s2[v][a1][c][b]: one item = the (v, c) fibres of the
    // rows a1 = k and N - 1 - k (N + 1 modal outputs per item, balanced as in modal_to_nodal)
    constexpr int NFC = NV * N, NK = (N + 1) / 2;
    for (int it = tid; it < NK * NFC; it += nt) {
      const int k = it / NFC, w = it - k * NFC, v = w / N, c = w - v * N;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int a1 = h == 0 ? k : N - 1 - k;
        if (h == 1 && a1 == k) break;
        const int prs = a1 * N - a1 * (a1 - 1) / 2;
        fiberK_n<N, true>(T.p2 + a1 * N * psi_np<N>(), N - a1, t2 + ((v * N + a1) * N + c) * N, 1,
                          t1 + (v * NPAIR + prs) * N + c, N);
      }
    }
    __syncthreads();
    // u[v][off(pr)+a3] = sum_c psi3[s][a3][c] s1[v][pr][c]; one (pr, v) fibre per item
    for (int it = tid; it < NPAIR * NV; it += nt) {
      const int pr = it / NV, v = it - pr * NV;
      const int sdeg = T.pa1[pr] + T.pa2[pr];
      fiberK_n<N, true>(T.p3 + sdeg * N * psi_np<N>(), N - sdeg, t1 + (v * NPAIR + pr) * N, 1, um + v * Np + T.poff[pr], 1);
    }
    __syncthreads();
  }
  (void)P;
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
// K1: entropy projection and traces (persistent: two CTAs per SM loop over elements)
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Slim K1 (experiment, off: ES_K1_SLIM=1 enables it for tetrahedra at N = 9): the shared-memory
// footprint cut from 111 KB to 72 KB so that three
// CTAs of 256 threads share an SM instead of two of 384 -- K1 is barrier-bound (one element's
// transform steps give ~200-400 work items between barriers), and a third element in flight hides
// more of it.  The facet values alias the second transform buffer, W J~ and W / J~ are read from
// global memory where they are used, and the psi2 / psi3 tables come from a padded global copy (L1).
#ifndef ES_K1_SLIM
#define ES_K1_SLIM 0  // measured slower at C5: 19.7 vs 17.9 ms per RHS
#endif
template <int DIM, int N>
__host__ __device__ constexpr bool k1_slim() {
  return ES_K1_SLIM && DIM == 3 && N == 9;
}
template <int DIM, int N>
struct ProjSmem {
  using S = Sz<DIM, N>;
  static constexpr bool SLIM = k1_slim<DIM, N>();
  static constexpr int ev(int x) { return (x + 1) & ~1; }
  static constexpr int XB = S::NC * S::Nq;            // nodal buffer
  static constexpr int T2B = S::NC * S::Nq;           // second transform buffer
  static constexpr int FWB = SLIM ? 0 : S::NC * S::NF;  // facet values (slim: in T2 after the facet-4 scratch)
  static constexpr int UMB = S::NC * S::Np;           // modal work buffer
  static constexpr int INB = S::NC * S::Np + (SLIM ? 0 : 2 * S::Nq);  // prefetched input: u~ (, W J~, W / J~)
  static constexpr int TBB = 3 * N + N * N;           // lL, lR, l3L, lint4
  static constexpr int o_x = 0, o_t2 = ev(o_x + XB), o_fw = SLIM ? o_t2 + ev(S::NC * N * N) : ev(o_t2 + T2B),
                       o_um = ev(o_t2 + T2B + FWB), o_in = ev(o_um + UMB), o_tb = ev(o_in + INB), o_ps = ev(o_tb + TBB),
                       total = o_ps + (SLIM ? 0 : psi_smem_doubles<DIM, N>());
  static_assert(S::NC * N * N <= T2B, "facet-4 scratch");
  static_assert(!SLIM || ev(S::NC * N * N) + S::NC * S::NF <= T2B, "slim: facet values fit behind the facet-4 scratch");
};
template <int DIM, int N>
__host__ __device__ constexpr int k1_threads() {
  return k1_slim<DIM, N>() ? 256 : Sz<DIM, N>::NT;
}

template <int DIM, int N>
__host__ __device__ constexpr size_t project_smem_doubles() {
  return ProjSmem<DIM, N>::total;
}

// resident CTAs per SM the register budget is sized for: about 20 warps per SM where shared memory
// allows (small elements have small CTAs), at least 2
template <int DIM, int N>
__host__ __device__ constexpr int k1_min_blocks() {
  constexpr int smem_fit = (227 * 1024) / (int)(project_smem_doubles<DIM, N>() * 8 + 1024);
  constexpr int want = k1_slim<DIM, N>() ? 3 : 20 / (Sz<DIM, N>::NT / 32);
  constexpr int b = want < smem_fit ? want : smem_fit;
  return b < 2 ? 2 : b;
}

template <int DIM, int N>
__global__ void __launch_bounds__(k1_threads<DIM, N>(), k1_min_blocks<DIM, N>()) project_kernel(DevRef R, ProjArgs A) {
  pdl_wait();
  PDL_TRIGGER();
  using S = Sz<DIM, N>;
  using L = ProjSmem<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf;
#ifndef ES_K1_PB
#define ES_K1_PB 1
#endif
  // nodes per thread and round in the pointwise phases: 2 measured slower than 1 (C5 K1 18.15 vs 17.29 ms:
  // registers, not latency, limit these phases)
  constexpr int PB = ES_K1_PB;
  extern __shared__ __align__(16) double sm[];
  double* X = sm + L::o_x;    // [NC][Nq]
  double* T2 = sm + L::o_t2;  // [NC][Nq]
  double* FW = sm + L::o_fw;  // [NC][NF]
  double* um = sm + L::o_um;  // [NC][Np]
  double* uin = sm + L::o_in;  // [NC][Np] u~, then W J~ [Nq], W / J~ [Nq] (not slim)
  const double* wj = uin + NC * Np;
  const double* wjinv = wj + Nq;
  double* tlL = sm + L::o_tb;
  double* tlR = tlL + N;
  double* tl3 = tlR + N;
  double* tli4 = tl3 + N;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double g = A.gamma, gm1 = g - 1.0, gm1inv = 1.0 / gm1, i1mg = 1.0 / (1.0 - g);
  auto elem_of = [&](int64_t idx) { return A.elem_list ? A.elem_list[idx] : idx; };
  // asynchronous copies (cp.async) of one element's inputs into uin / wj / wjinv
  auto prefetch = [&](int64_t e) {
    const double* src = A.u + (size_t)e * NC * Np;
    for (int k = tid; k < NC * Np; k += nt) cp_async8(uin + k, src + k);
    if constexpr (!L::SLIM) {
      const double* gv = A.geo_vol + (size_t)e * S::GVS + S::NG * Nq;
      for (int k = tid; k < 2 * Nq; k += nt) cp_async8(uin + NC * Np + k, gv + k);
    }
    cp_async_commit();
  };
  if ((int64_t)blockIdx.x < A.n_elem) prefetch(elem_of(blockIdx.x));
  const PsiS T = L::SLIM ? psi_tables<DIM, N>(const_cast<double*>(R.psig)) : stage_psi<DIM, N>(R, sm + L::o_ps);
  for (int k = tid; k < N; k += nt) {
    tlL[k] = R.lL[k];
    tlR[k] = R.lR[k];
    if constexpr (DIM == 3) tl3[k] = R.l3L[k];
  }
  if constexpr (DIM == 3)
    for (int k = tid; k < N * N; k += nt) tli4[k] = R.lint4[k];
  int bad = 0;
#pragma unroll 1
  for (int64_t idx = blockIdx.x; idx < A.n_elem; idx += gridDim.x) {
    const int64_t e = elem_of(idx);
    auto stamp = [&](int q) {
      #ifdef ES_STAMPS  // diagnostics build only (tools/build.py with ES_STAMPS=1)
    if (A.dbg && tid == 0 && idx < 4096) A.dbg[idx * 16 + q] = clock64();
#else
    (void)q;
#endif
    };
    stamp(0);
    if constexpr (L::SLIM) {  // W J~ and W / J~ straight from global memory
      wj = A.geo_vol + (size_t)e * S::GVS + S::NG * Nq;
      wjinv = wj + Nq;
    }
    cp_async_wait_all();
    __syncthreads();
    stamp(1);
    // u = V u~ (ping-pong X / T2; 3D writes its first scratch into the output buffer)
    if constexpr (DIM == 3)
      modal_to_nodal<DIM, N, NC>(T, uin, X, X, T2);
    else
      modal_to_nodal<DIM, N, NC>(T, uin, X, T2, nullptr);
    stamp(2);
    // W J~ W(u)   (App. B formulas, R7): PB nodes per thread as independent straight-line streams
    // (branch-free log, fastmath.cuh)
    for (int i0 = tid; i0 < Nq; i0 += PB * nt) {
      double U[PB][NC], ir[PB], pp[PB], lr[PB], lp[PB];
      int ii[PB];
      bool nanj[PB] = {};
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        const int i = i0 + j * nt;
        ii[j] = i < Nq ? i : i0;  // an absent node recomputes the first one and stores nothing
#pragma unroll
        for (int v = 0; v < NC; ++v) U[j][v] = X[v * Nq + ii[j]];
      }
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        if (!(U[j][0] > 0.0 && U[j][0] < 1e300)) {
          bad = 1;
          nanj[j] = true;
          U[j][0] = 1.0;
        }
        ir[j] = es_fm_rcp(U[j][0]);
        double ke = 0.0;
#pragma unroll
        for (int m = 0; m < DIM; ++m) {
          const double vm = U[j][1 + m] * ir[j];  // velocity
          ke += vm * U[j][1 + m];
          U[j][1 + m] = vm;
        }
        pp[j] = gm1 * (U[j][DIM + 1] - 0.5 * ke);
        if (!(pp[j] > 0.0 && pp[j] < 1e300)) {
          bad = 1;
          nanj[j] = true;
          pp[j] = 1.0;  // keep the branch-free log inside its domain; the result is set to NaN below
        }
      }
#pragma unroll
      for (int j = 0; j < PB; ++j) lr[j] = es_log_pos(U[j][0]);
#pragma unroll
      for (int j = 0; j < PB; ++j) lp[j] = nanj[j] ? __longlong_as_double(0x7ff8000000000000LL) : es_log_pos(pp[j]);
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        const double s = lp[j] - g * lr[j], beta = U[j][0] * es_fm_rcp(pp[j]);
        double v2 = 0.0;
#pragma unroll
        for (int m = 0; m < DIM; ++m) v2 += U[j][1 + m] * U[j][1 + m];
        if (j == 0 || i0 + j * nt < Nq) {
          const int i = ii[j];
          const double w = wj[i];
          X[0 * Nq + i] = w * ((g - s) * gm1inv - 0.5 * beta * v2);
#pragma unroll
          for (int m = 0; m < DIM; ++m) X[(1 + m) * Nq + i] = w * beta * U[j][1 + m];
          X[(DIM + 1) * Nq + i] = -w * beta;
        }
      }
    }
    __syncthreads();
    stamp(3);
    if constexpr (DIM == 3) {
      nodal_to_modal<DIM, N, NC>(T, X, um, X, T2);
      stamp(4);
      modal_to_nodal<DIM, N, NC>(T, um, X, X, T2);
      stamp(5);
      nodal_to_modal<DIM, N, NC>(T, X, um, X, T2, wjinv);  // w~, W / J~ fused into the loads
    } else {
      nodal_to_modal<DIM, N, NC>(T, X, um, T2, nullptr);
      stamp(4);
      modal_to_nodal<DIM, N, NC>(T, um, X, T2, nullptr);
      stamp(5);
      nodal_to_modal<DIM, N, NC>(T, X, um, T2, nullptr, wjinv);
    }
    stamp(7);
    // the prefetched inputs are consumed: the next element's copies overlap the rest
    if (idx + gridDim.x < A.n_elem) prefetch(elem_of(idx + gridDim.x));
    if (A.wt)
      for (int k = tid; k < NC * Np; k += nt) A.wt[(size_t)e * NC * Np + k] = um[k];
    if constexpr (DIM == 3)  // w = V w~
      modal_to_nodal<DIM, N, NC>(T, um, X, X, T2);
    else
      modal_to_nodal<DIM, N, NC>(T, um, X, T2, nullptr);
    stamp(8);
    // w_f = R^(z) w along lines; facet 4 (3D) contracts eta3 first: y[a][b] = sum_c l3(c) w
    if constexpr (DIM == 3) {
      double* y = T2;  // [NC][N(b)][N(a)]
      for (int it = tid; it < NC * N * N; it += nt) {
        const int v = it / (N * N), ab = it - v * N * N;
        const double* x = X + v * Nq + ab;
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < N; ++c) s = fma(tl3[c], x[N * N * c], s);
        y[it] = s;
      }
      __syncthreads();
    }
    if constexpr (DIM == 3) {
      // warp tasks (variable, kind, 32-node part): kind 0 = facet 1 (along eta2), kind 1 = facets 2 and 3
      // (both along eta1, sharing the line's loads), kind 2 = facet 4 (eta2 contraction of y); the kind
      // is warp-uniform, so the index arithmetic is a few integer instructions per item
      constexpr int PARTS = (Nqf + 31) / 32;
      const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
      for (int task = warp; task < NC * 3 * PARTS; task += nw) {
        const int v = task / (3 * PARTS), rr = task - v * 3 * PARTS, kind = rr / PARTS, f = (rr - kind * PARTS) * 32 + lane;
        if (f < Nqf) {
          const int f1 = f % N, f2 = f / N;
          double* fw = FW + v * NF + f;
          if (kind == 0) {
            const double* x = X + v * Nq + f1 + N * N * f2;
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b) s = fma(tlL[b], x[N * b], s);
            fw[0] = s;
          } else if (kind == 1) {
            const double* x = X + v * Nq + N * f1 + N * N * f2;
            double sR = 0.0, sL = 0.0;
#pragma unroll
            for (int a = 0; a < N; ++a) {
              const double xa = x[a];
              sR = fma(tlR[a], xa, sR);
              sL = fma(tlL[a], xa, sL);
            }
            fw[Nqf] = sR;
            fw[2 * Nqf] = sL;
          } else {
            const double* y = T2 + v * N * N + f1;
            const double* l = tli4 + f2 * N;
            double s = 0.0;
#pragma unroll
            for (int b = 0; b < N; ++b) s = fma(l[b], y[N * b], s);
            fw[3 * Nqf] = s;
          }
        }
      }
    } else {
      for (int it = tid; it < NC * NF; it += nt) {
        const int v = it / NF, fz = it - v * NF, z = fz / Nqf, f = fz - z * Nqf;
        const double* x = X + v * Nq;
        double s = 0.0;
        if (z == 0) {
#pragma unroll
          for (int b = 0; b < N; ++b) s = fma(tlL[b], x[f + N * b], s);
        } else {
          const double* l = z == 1 ? tlR : tlL;
#pragma unroll
          for (int a = 0; a < N; ++a) s = fma(l[a], x[a + N * f], s);
        }
        FW[it] = s;
      }
    }
    __syncthreads();
    stamp(9);
    // entropy-projected conservative variables U(w) -> stored as primitive (rho, v, p) and
    // beta = rho / p = -w_last (App. B); the spread of rho and beta over the element's volume and
    // facet nodes decides the all-Taylor flag ((max - min) < 0.0099 (max + min) for both implies
    // f2 = ((x - y)/(x + y))^2 < 1e-4 for every pair, reading R5)
    double mm[4] = {1e300, -1e300, 1e300, -1e300};  // rho min, max, beta min, max
    // PB nodes per thread as independent straight-line streams (branch-free log / exp, fastmath.cuh)
    for (int i0 = tid; i0 < Nq + NF; i0 += PB * nt) {
      double w[PB][NC], b[PB], ib[PB], arg[PB], r[PB];
      bool nanj[PB] = {};
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        const int i = (j == 0 || i0 + j * nt < Nq + NF) ? i0 + j * nt : i0;  // an absent node repeats the first
        if (i < Nq) {
#pragma unroll
          for (int v = 0; v < NC; ++v) w[j][v] = X[v * Nq + i];
        } else {
#pragma unroll
          for (int v = 0; v < NC; ++v) w[j][v] = FW[v * NF + (i - Nq)];
        }
      }
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        b[j] = -w[j][DIM + 1];
        if (!(b[j] > 0.0 && b[j] < 1e300)) {
          nanj[j] = true;
          b[j] = 1.0;
        }
        ib[j] = es_fm_rcp(b[j]);
        double v2 = 0.0;
#pragma unroll
        for (int m = 0; m < DIM; ++m) {
          w[j][1 + m] *= ib[j];  // velocity
          v2 += w[j][1 + m] * w[j][1 + m];
        }
        arg[j] = g - gm1 * (w[j][0] + 0.5 * b[j] * v2);  // s
      }
#pragma unroll
      for (int j = 0; j < PB; ++j) arg[j] = (arg[j] + es_log_pos(b[j])) * i1mg;
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        if (!(fabs(arg[j]) < 600.0)) {
          nanj[j] = true;
          arg[j] = 0.0;
        }
        r[j] = es_exp(arg[j]);  // (b e^s)^(1/(1-g))
      }
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        if (nanj[j]) {  // inadmissible projected state: flag it and let NaN propagate (as log / exp would)
          bad = 1;
          r[j] = b[j] = ib[j] = __longlong_as_double(0x7ff8000000000000LL);
        }
        if (j == 0 || i0 + j * nt < Nq + NF) {
          const int i = i0 + j * nt;
          const double ph = 0.5 * (r[j] * ib[j]);  // p / 2: the flux uses half pressures (exact scaling)
          if (i < Nq) {
            double* o = A.prim + (size_t)e * S::PRS + i;
            o[0] = r[j];
#pragma unroll
            for (int m = 0; m < DIM; ++m) o[(1 + m) * Nq] = w[j][1 + m];
            o[(DIM + 1) * Nq] = ph;
            o[(DIM + 2) * Nq] = b[j];
          } else {
            const int fz = i - Nq, z = fz / Nqf, f = fz - z * Nqf;
            double* o = A.trace + (((size_t)e * S::Nf + z) * NC) * Nqf + f;
            o[0] = r[j];
#pragma unroll
            for (int m = 0; m < DIM; ++m) o[(1 + m) * Nqf] = w[j][1 + m];
            o[(DIM + 1) * Nqf] = ph;
          }
          mm[0] = r[j] < mm[0] ? r[j] : mm[0];
          mm[1] = r[j] > mm[1] ? r[j] : mm[1];
          mm[2] = b[j] < mm[2] ? b[j] : mm[2];
          mm[3] = b[j] > mm[3] ? b[j] : mm[3];
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double t0 = __shfl_xor_sync(0xffffffffu, mm[0], o), t1 = __shfl_xor_sync(0xffffffffu, mm[1], o);
      const double t2 = __shfl_xor_sync(0xffffffffu, mm[2], o), t3 = __shfl_xor_sync(0xffffffffu, mm[3], o);
      mm[0] = t0 < mm[0] ? t0 : mm[0];
      mm[1] = t1 > mm[1] ? t1 : mm[1];
      mm[2] = t2 < mm[2] ? t2 : mm[2];
      mm[3] = t3 > mm[3] ? t3 : mm[3];
    }
    __shared__ double red_mm[16][4];  // NT <= 512
    if ((tid & 31) == 0)
#pragma unroll
      for (int q = 0; q < 4; ++q) red_mm[tid >> 5][q] = mm[q];
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nt / 32; ++w) {
        mm[0] = red_mm[w][0] < mm[0] ? red_mm[w][0] : mm[0];
        mm[1] = red_mm[w][1] > mm[1] ? red_mm[w][1] : mm[1];
        mm[2] = red_mm[w][2] < mm[2] ? red_mm[w][2] : mm[2];
        mm[3] = red_mm[w][3] > mm[3] ? red_mm[w][3] : mm[3];
      }
      const bool taylor = (mm[1] - mm[0]) < 0.0099 * (mm[1] + mm[0]) && (mm[3] - mm[2]) < 0.0099 * (mm[3] + mm[2]);
      A.prim[(size_t)e * S::PRS + (NC + 1) * Nq] = taylor ? 1.0 : 0.0;
    }
    stamp(10);
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
  extern __shared__ __align__(16) double sm[];
  constexpr int o_um = (NC * Nq + 1) & ~1, o_t1 = (o_um + NC * Np + 1) & ~1, o_t2 = (o_t1 + t1_size<DIM, N>() + 1) & ~1,
                o_ps = (o_t2 + t2_size<DIM, N>() + 1) & ~1;
  double* X = sm;
  double* um = sm + o_um;
  double* T1 = sm + o_t1;
  double* T2 = sm + o_t2;
  const PsiS T = stage_psi<DIM, N>(R, sm + o_ps);
  int64_t e = blockIdx.x;
  for (int it = threadIdx.x; it < NC * Nq; it += blockDim.x) {
    int v = it / Nq, i = it % Nq;
    X[it] = __ldg(&R.Wvol[i]) * un[((size_t)e * Nq + i) * NC + v];
  }
  __syncthreads();
  nodal_to_modal<DIM, N, NC>(T, X, um, T1, T2);
  for (int k = threadIdx.x; k < NC * Np; k += blockDim.x) um_out[(size_t)e * NC * Np + k] = um[k];
}

// modal -> nodal evaluation u = V u~ at the volume nodes, [ne][NC][Np] -> [ne][Nq][NC] (output)
template <int DIM, int N>
__global__ void __launch_bounds__(Sz<DIM, N>::NT) eval_nodal_kernel(DevRef R, int64_t ne, const double* um_in,
                                                                 double* un) {
  using S = Sz<DIM, N>;
  constexpr int NC = S::NC, Nq = S::Nq, Np = S::Np;
  extern __shared__ __align__(16) double sm[];
  constexpr int o_um = (NC * Nq + 1) & ~1, o_t1 = (o_um + NC * Np + 1) & ~1, o_t2 = (o_t1 + t1_size<DIM, N>() + 1) & ~1,
                o_ps = (o_t2 + t2_size<DIM, N>() + 1) & ~1;
  double* X = sm;
  double* um = sm + o_um;
  double* T1 = sm + o_t1;
  double* T2 = sm + o_t2;
  const PsiS T = stage_psi<DIM, N>(R, sm + o_ps);
  const int64_t e = blockIdx.x;
  for (int k = threadIdx.x; k < NC * Np; k += blockDim.x) um[k] = um_in[(size_t)e * NC * Np + k];
  __syncthreads();
  modal_to_nodal<DIM, N, NC>(T, um, X, T1, T2);
  for (int it = threadIdx.x; it < NC * Nq; it += blockDim.x) {
    const int v = it / Nq, i = it - v * Nq;
    un[((size_t)e * Nq + i) * NC + v] = X[it];
  }
}

template <int DIM, int N>
__host__ __device__ constexpr size_t projnodal_smem_doubles() {
  using S = Sz<DIM, N>;
  return (size_t)S::NC * S::Nq + (size_t)S::NC * S::Np + t1_size<DIM, N>() + t2_size<DIM, N>() + 4 +
         psi_smem_doubles<DIM, N>();
}

}  // namespace esb
