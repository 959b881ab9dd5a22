// psi_const.cuh -- the PKD sum-factorisation tables of one degree in constant memory (read as
// warp-uniform operands) and the even-odd form of the psi1 contractions (product code, 3D paths).
// Each translation unit that uses c_psi<N> holds its own copy; the library uploads it per unit
// (upload_psi_3d, upload_psi_3d_k1).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <utility>

namespace esb {

// Programmatic dependent launch (PDL): the kernels of one RK stage chain (K1 -> K2 -> K3 -> K1 ...) are
// launched with cudaLaunchAttributeProgrammaticStreamSerialization (launch_pdl), so a kernel's grid is
// scheduled while its predecessor drains.  Every such kernel calls pdl_wait() (griddepcontrol.wait:
// blocks until the predecessor grid has completed and its memory is visible) unconditionally before
// touching any buffer another kernel writes or reads, and pdl_trigger() (launch_dependents) so that its
// own successor may be scheduled as soon as all of its CTAs are running.  Both are no-ops for a normal
// launch.  The chain is transitive: each kernel's completion implies its predecessor's.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#ifndef ES_PDL_TRIGGER  // explicit early trigger (1) or the implicit one at CTA exit (0)
#define ES_PDL_TRIGGER 0
#endif
#define PDL_TRIGGER() \
  do {                \
    if (ES_PDL_TRIGGER) pdl_trigger(); \
  } while (0)

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

// host: launch with the PDL attribute (see pdl_wait)
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  static const bool off = std::getenv("ES_NO_PDL") != nullptr;  // measurement switch: plain launches
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace esb
