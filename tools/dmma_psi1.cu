// dmma_psi1.cu -- the psi1 step of the sum-factorised transforms (u[a] = sum_a1 psi1[a1][a] t2[a1], N = 9)
// on a batch of fibres in shared memory, as (a) DFMA in the even-odd form with constant-memory tables
// (what K1 / K3 run) and (b) DMMA mma.sync.m8n8k4.f64 with the fibres on M (no M padding) and the
// table on B held in registers (k padded 9 -> 12, n padded 9 -> 16).  Measures fibres/s of each; the
// DMMA and DFMA pipes are the same (tools/fp64_pipes.cu), so the padding decides.  Prints JSON lines.
#include <cuda_runtime.h>

#include <cstdio>

#include "psi_const.cuh"

using namespace esb;
constexpr int N = 9, FPB = 512;  // fibres per block-iteration (smem [FPB][10])

__global__ void __launch_bounds__(256) dfma_eo(double* out, int reps) {
  __shared__ double x[FPB * 10];
  for (int k = threadIdx.x; k < FPB * 10; k += blockDim.x) x[k] = 1.0 + 1e-3 * (k % 17);
  __syncthreads();
  double acc = 0.0;
  for (int r = 0; r < reps; ++r) {
    for (int f = threadIdx.x; f < FPB; f += blockDim.x) {
      double in[N], o[N];
#pragma unroll
      for (int a = 0; a < N; ++a) in[a] = x[f * 10 + a];
      psi1_apply_eo<N>(in, o);
#pragma unroll
      for (int a = 0; a < N; ++a) x[f * 10 + a] = o[a] * 0.5;
    }
    __syncthreads();
  }
  acc = x[threadIdx.x];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256) dmma(double* out, int reps, const double* __restrict__ tab) {
  __shared__ double x[FPB * 10];
  for (int k = threadIdx.x; k < FPB * 10; k += blockDim.x) x[k] = 1.0 + 1e-3 * (k % 17);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  // B fragments: B[k][n] = psi1[k0 + (lane & 3)][n0 + (lane >> 2)] for 3 k-steps x 2 n-tiles
  double b[3][2];
#pragma unroll
  for (int ks = 0; ks < 3; ++ks)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int k = ks * 4 + (lane & 3), n = nt * 8 + (lane >> 2);
      b[ks][nt] = (k < N && n < N) ? tab[k * N + n] : 0.0;
    }
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    for (int f0 = warp * 8; f0 < FPB; f0 += nw * 8) {
      const int row = f0 + (lane >> 2);
      double c[2][2] = {{0, 0}, {0, 0}};
#pragma unroll
      for (int ks = 0; ks < 3; ++ks) {
        const int k = ks * 4 + (lane & 3);
        const double a = k < N ? x[row * 10 + k] : 0.0;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(c[nt][0]), "+d"(c[nt][1])
                       : "d"(a), "d"(b[ks][nt]));
      }
      __syncwarp();
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const int col = nt * 8 + 2 * (lane & 3) + q;
          if (col < N) x[(f0 + (lane >> 2)) * 10 + col] = c[nt][q] * 0.5;
        }
      __syncwarp();
    }
    __syncthreads();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x[threadIdx.x];
}

int main() {
  PsiC<N> h;
  double tab[N * N];
  for (int a1 = 0; a1 < N; ++a1)
    for (int a = 0; a < N; ++a) tab[a1 * N + a] = h.p1[a1 * N + a] = ((a1 % 2) && a > N / 2 ? -1 : 1) * 0.1 * (1 + a1);
  for (int k = 0; k < N * N * N; ++k) h.p2[k] = h.p3[k] = 0.0;
  cudaMemcpyToSymbol(c_psi<N>, &h, sizeof(h));
  double *out, *dt;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  cudaMalloc(&dt, sizeof(tab));
  cudaMemcpy(dt, tab, sizeof(tab), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 2, reps = 400;
  for (int v = 0; v < 2; ++v) {
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(e0);
      if (v == 0)
        dfma_eo<<<blocks, 256>>>(out, reps);
      else
        dmma<<<blocks, 256>>>(out, reps, dt);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fibres = (double)blocks * FPB * reps;
    printf("{\"variant\": \"%s\", \"ms\": %.3f, \"fibres_per_s\": %.4g, \"useful_tflops\": %.2f, \"err\": \"%s\"}\n",
           v == 0 ? "dfma_even_odd" : "dmma_m8n8k4", ms, fibres / (ms * 1e-3), 2.0 * 81 * fibres / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
