// Accuracy of the flux kernel's reciprocal (rhs2.cuh rcp_nr): the rcp.approx.ftz.f64 seed refined by
// one cubic step r (1 + e + e^2), e = 1 - s r, against the correctly rounded 1/s, over 2^26 arguments
// spread over [2^-20, 2^20].  Prints the largest error in units of the last place.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ double rcp_c3(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  const double e = fma(-s, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__global__ void k(unsigned long long* worst, double* seed_err) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t h = i * 0x9E3779B97F4A7C15ull;
  h ^= h >> 29;
  double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);  // [0, 1)
  double s = exp2(-20.0 + 40.0 * u);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  double ex = __drcp_rn(s);
  double rel = fabs(r - ex) / ex;
  unsigned long long b = __double_as_longlong(rel);
  atomicMax((unsigned long long*)seed_err, b);
  double c = rcp_c3(s);
  long long ulp = __double_as_longlong(c) - __double_as_longlong(ex);
  atomicMax(worst, (unsigned long long)(ulp < 0 ? -ulp : ulp));
}
int main() {
  unsigned long long* w;
  double* se;
  cudaMallocManaged(&w, 8);
  cudaMallocManaged(&se, 8);
  *w = 0;
  *se = 0.0;
  k<<<1 << 18, 256>>>(w, se);
  cudaDeviceSynchronize();
  printf("{\"seed_max_rel_err\": %.3e, \"cubic_step_max_ulp\": %llu}\n", *se, *w);
  return 0;
}
