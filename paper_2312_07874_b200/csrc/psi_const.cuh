// psi_const.cuh -- the PKD sum-factorisation tables of one degree in constant memory (read as
// warp-uniform operands) and the even-odd form of the psi1 contractions (product code, 3D paths).
// Each translation unit that uses c_psi<N> holds its own copy; the library uploads it per unit
// (upload_psi_3d, upload_psi_3d_k1).
#pragma once
#include <cuda_runtime.h>

namespace esb {

template <int N>
struct PsiC {
  double p1[N * N];      // psi1[a1][a]
  double p2[N * N * N];  // psi2[a1][a2][b]
  double p3[N * N * N];  // psi3[s][a3][c]
};
template <int N>
__constant__ PsiC<N> c_psi;

// even-odd (parity) form of the psi1 contractions: the Legendre nodes are symmetric (eta_{N-1-a} =
// -eta_a) and psi1^{a1} has the parity of a1, so psi1[a1][N-1-a] = (-1)^{a1} psi1[a1][a] and
//   u[a] = ue[a] + uo[a], u[N-1-a] = ue[a] - uo[a],  ue = even-a1 sums, uo = odd-a1 sums, a < N/2
// halves the multiply-adds of the largest sum-factorisation step (checked on the host at setup)
template <int N>
__device__ __forceinline__ void psi1_apply_eo(const double* t2, double* u) {  // u[a] = sum_a1 psi1[a1][a] t2[a1]
  constexpr int H = N / 2, M = N % 2;
#pragma unroll
  for (int a = 0; a < H + M; ++a) {
    double ue = 0.0, uo = 0.0;
#pragma unroll
    for (int a1 = 0; a1 < N; a1 += 2) ue = fma(c_psi<N>.p1[a1 * N + a], t2[a1], ue);
    if (a < H) {
#pragma unroll
      for (int a1 = 1; a1 < N; a1 += 2) uo = fma(c_psi<N>.p1[a1 * N + a], t2[a1], uo);
      u[a] = ue + uo;
      u[N - 1 - a] = ue - uo;
    } else {
      u[a] = ue;  // middle node: the odd functions vanish there
    }
  }
}
template <int N>
__device__ __forceinline__ void psi1T_apply_eo(const double* y, double* s2) {  // s2[a1] = sum_a psi1[a1][a] y[a]
  constexpr int H = N / 2, M = N % 2;
  double yp[H + M], ym[H > 0 ? H : 1];
#pragma unroll
  for (int a = 0; a < H; ++a) {
    yp[a] = y[a] + y[N - 1 - a];
    ym[a] = y[a] - y[N - 1 - a];
  }
  if (M) yp[H] = y[H];
#pragma unroll
  for (int a1 = 0; a1 < N; ++a1) {
    double t = 0.0;
    if (a1 % 2 == 0) {
#pragma unroll
      for (int a = 0; a < H + M; ++a) t = fma(c_psi<N>.p1[a1 * N + a], yp[a], t);
    } else {
#pragma unroll
      for (int a = 0; a < H; ++a) t = fma(c_psi<N>.p1[a1 * N + a], ym[a], t);
    }
    s2[a1] = t;
  }
}

}  // namespace esb
