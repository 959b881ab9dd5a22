// fp64_pipes.cu -- do DFMA (FP64 pipe) and DMMA (mma.sync.m8n8k4.f64) share one execution pipe on
// the B200?  Times the same per-warp work as (a) all warps DFMA, (b) all warps DMMA, (c) half the
// warps of every CTA DFMA and half DMMA.  If (c) takes about max(a, b)/2 ... i.e. the two halves
// overlap, the pipes are separate and sum-factorised transforms on DMMA could run beside the
// flux arithmetic on DFMA.  Prints one JSON object.  (Design input for DESIGN.md section 5.)
#include <cuda_runtime.h>

#include <cstdio>

template <int MODE>  // 0 DFMA, 1 DMMA, 2 even warps DFMA / odd warps DMMA
__global__ void mix(double* out, int iters, double a, double b) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = MODE == 1 || (MODE == 2 && (warp & 1));
  double s = 0.0;
  if (do_mma) {
    double c[8][2];
    double x = 1.0 + threadIdx.x * 1e-3, y = 0.5;
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
    // per iteration: 8 DMMA = 8 * 256 MACs per warp = 64 MACs per lane
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[k][0]), "+d"(c[k][1])
                     : "d"(x), "d"(y));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  } else {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    // per iteration: 64 DFMA per lane
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 4 * 512);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    return best;
  };
  const int blocks = sms * 4, threads = 512, iters = 4096;
  const double macs = 64.0 * iters * blocks * threads;  // MACs per lane per launch, all lanes
  float t0 = timeit([&] { mix<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
  float t1 = timeit([&] { mix<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
  float t2 = timeit([&] { mix<2><<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
  printf("{\"sms\": %d, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f, \"mixed_ms\": %.3f, \"dfma_tflops\": %.2f, "
         "\"dmma_tflops\": %.2f, \"mixed_tflops\": %.2f, \"separate_pipes\": %s}\n",
         sms, t0, t1, t2, 2 * macs / (t0 * 1e-3) / 1e12, 2 * macs / (t1 * 1e-3) / 1e12,
         2 * macs / (t2 * 1e-3) / 1e12, (t2 < 0.75 * (t0 < t1 ? t1 : t0)) ? "true" : "false");
  return 0;
}
