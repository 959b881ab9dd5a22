// fp64_micro.cu -- FP64 microbenchmarks on the B200 (roofline denominators and design inputs,
// DESIGN.md section 5): DFMA throughput, DFMA dependent-chain latency, MUFU.RCP64H + Newton
// latency, and DMMA (mma.sync.m8n8k4.f64) throughput.  Prints one JSON object.
#include <cuda_runtime.h>

#include <cstdio>

__global__ void dfma_tp(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 64; ++r) x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void rcp_lat(double* out, long long* cyc, int iters, double s0) {
  double x = s0 + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double rr;
      asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(rr) : "d"(x));
      x = rr + 1.5;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void dmma_tp(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * sms * 8 * 256);
  cudaMalloc(&cyc, sizeof(long long));
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
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float ms = timeit([&] { dfma_tp<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); });
  double dfma_tflops = 2.0 * 8 * 16 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
  long long h;
  dfma_lat<<<1, 32>>>(out, cyc, 1024, 0.999999, 1e-7);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double lat_dfma = (double)h / (1024.0 * 64);
  rcp_lat<<<1, 32>>>(out, cyc, 1024, 1.25);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double lat_rcp_add = (double)h / (1024.0 * 16);
  float ms2 = timeit([&] { dmma_tp<<<blocks, threads>>>(out, 2048); });
  double dmma_tflops = 2.0 * 256 * 8 * 2048.0 * blocks * (threads / 32) / (ms2 * 1e-3) / 1e12;
  printf("{\"sms\": %d, \"clock_khz_attr\": %d, \"dfma_tflops\": %.3f, \"dfma_latency_cyc\": %.2f, "
         "\"rcp64h_plus_dadd_latency_cyc\": %.2f, \"dmma_m8n8k4_tflops\": %.3f}\n",
         sms, clk, dfma_tflops, lat_dfma, lat_rcp_add, dmma_tflops);
  return 0;
}
