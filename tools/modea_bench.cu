// modea_bench.cu -- isolates the mode-A c-slab transform of K3 (xform3.cuh): V steps 2-3, W/J~
// scaling, V^T steps 1-2 of one (element, variable, c) lane, repeated over shared-memory data, to
// measure its FP64 throughput apart from global loads, barriers and the B-mode phases.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -I paper_2312_07874_b200/csrc tools/modea_bench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "xform3.cuh"

using namespace esb;

template <int N, int VAR, int MINB, int NTH = 192>
__global__ void __launch_bounds__(NTH, MINB) bench_mid(double* out, int reps, int zero) {
  using Z = X3<N>;
  extern __shared__ __align__(16) double sm[];
  const int E = NTH / (5 * N);
  double* S = sm;                  // [E*5][SEV]
  double* W = S + E * 5 * Z::SEV;  // [E][Nq]
  const int tid = threadIdx.x;
  for (int k = tid; k < E * 5 * Z::SEV; k += blockDim.x) S[k] = 1.0 + 1e-3 * (k % 17);
  for (int k = tid; k < E * Z::Nq; k += blockDim.x) W[k] = 0.5 + 1e-3 * (k % 13);
  __syncthreads();
  const bool act = tid < 5 * E * N;
  const int ev = act ? tid / N : 0, c = act ? tid - ev * N : 0, e = ev / 5;
  for (int r = 0; r < reps; ++r) {
    if constexpr (VAR == 2)
      modeA_mid<N>(S + ev * Z::SEV + c, W + e * Z::Nq + c, act);
    else
      modeA_mid_t1reg<N>(S + ev * Z::SEV + c, W + e * Z::Nq + c, act);
    __syncwarp();
  }
  if (tid == 0) out[blockIdx.x] = S[0];
}

int main() {
  constexpr int N = 9;
  using Z = X3<N>;
  std::vector<double> p1(N * N), p2(N * N * N), p3(N * N * N);
  for (int k = 0; k < N * N; ++k) p1[k] = 1e-2 * (k % 5);
  for (int k = 0; k < N * N * N; ++k) p2[k] = p3[k] = 1e-2 * (k % 3);
  PsiC<N> h;
  for (int k = 0; k < N * N; ++k) h.p1[k] = p1[k];
  for (int k = 0; k < N * N * N; ++k) h.p2[k] = h.p3[k] = p2[k];
  cudaMemcpyToSymbol(c_psi<N>, &h, sizeof(h));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 200;
  const char* names[3] = {"evenodd-168reg-192thr", "t1reg-224reg-288thr", "t1reg-255reg-256thr"};
  const int nths[3] = {192, 288, 256};
  for (int var = 0; var < 3; ++var) {
    auto k = var == 0 ? bench_mid<N, 2, 2, 192> : var == 1 ? bench_mid<N, 3, 1, 288> : bench_mid<N, 3, 1, 256>;
    const int nth = nths[var];
    const int E = nth / (5 * N);
    const size_t smem = (E * 5 * Z::SEV + E * Z::Nq + 4 + N * 46) * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int cps : {1, 2}) {
      if (var > 0 && cps > 1) continue;
      k<<<sms * cps, nth, smem>>>(out, 2, 0);
      cudaEventRecord(a);
      k<<<sms * cps, nth, smem>>>(out, reps, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      // MACs per lane per call: 2 (45 + 81) per b
      const double macs = (double)sms * cps * 5 * E * N * reps * N * 2.0 * (45 + 81);
      // tflops counts the plain sum-factorised multiply-adds (the even-odd form does fewer)
      printf("{\"variant\": \"%s\", \"ctas_per_sm\": %d, \"ms\": %.3f, \"tflops_equiv\": %.2f, \"err\": \"%s\"}\n",
             names[var], cps, ms, 2 * macs / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
