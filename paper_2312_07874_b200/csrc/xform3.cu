// xform3.cu -- instantiations of the batched tetrahedral weight-adjusted inverse K3 (xform3.cuh) for
// q = p = N-1 in [1, 8], its constant-memory PKD tables, and the W / J~ layout permutation.
#include <cuda_runtime.h>

#include "xform3.cuh"

namespace esb {

namespace {
constexpr int kMaxDev = 64;

template <int N>
cudaError_t upload_psi(const double* p1, const double* p2, const double* p3) {
  PsiC<N> h;
  for (int k = 0; k < N * N; ++k) h.p1[k] = p1[k];
  for (int k = 0; k < N * N * N; ++k) {
    h.p2[k] = p2[k];
    h.p3[k] = p3[k];
  }
  return cudaMemcpyToSymbol(c_psi<N>, &h, sizeof(h));
}

template <int N>
cudaError_t do_wadj(const WadjArgs& A, cudaStream_t st) {
  if (A.n_elem <= 0) return cudaSuccess;
  using Z = X3<N>;
  static bool attr[kMaxDev] = {};  // the >48 KB shared-memory opt-in is per device
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
  if (!attr[dev]) {
    e = cudaFuncSetAttribute(wadj3_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z::SMEM);
    if (e != cudaSuccess) return e;
    attr[dev] = true;
  }
  const int64_t grid = (A.n_elem + Z::E - 1) / Z::E;
  return launch_pdl(wadj3_kernel<N>, dim3((unsigned)grid), dim3(Z::NT), Z::SMEM, st, A);
}

template <int N>
cudaError_t do_perm(const double* geo_vol, int gvs, int row, int64_t ne, double* out, cudaStream_t st) {
  if (ne <= 0) return cudaSuccess;
  const int64_t n = ne * N * N * N;
  wjinv_permute_kernel<N><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(geo_vol, gvs, row, ne, out);
  return cudaGetLastError();
}
}  // namespace

#define ES_X3_CASES(F, ...)            \
  switch (n) {                         \
    case 2: return F<2>(__VA_ARGS__);  \
    case 3: return F<3>(__VA_ARGS__);  \
    case 4: return F<4>(__VA_ARGS__);  \
    case 5: return F<5>(__VA_ARGS__);  \
    case 6: return F<6>(__VA_ARGS__);  \
    case 7: return F<7>(__VA_ARGS__);  \
    case 8: return F<8>(__VA_ARGS__);  \
    case 9: return F<9>(__VA_ARGS__);  \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t upload_psi_3d(int n, const double* p1, const double* p2, const double* p3) {
  ES_X3_CASES(upload_psi, p1, p2, p3)
}
cudaError_t launch_wadj_3d(int n, const WadjArgs& A, cudaStream_t st) { ES_X3_CASES(do_wadj, A, st) }
cudaError_t launch_wjinv_permute_3d(int n, const double* geo_vol, int gvs, int row, int64_t ne, double* out,
                                    cudaStream_t st) {
  ES_X3_CASES(do_perm, geo_vol, gvs, row, ne, out, st)
}

}  // namespace esb
