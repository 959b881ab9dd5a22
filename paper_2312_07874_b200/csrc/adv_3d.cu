// adv_3d.cu -- instantiations of the linear-advection kernels (advect.cuh) for tetrahedra
#include "advect.cuh"

namespace esb {

template <int DIM, int N>
static cudaError_t do_adv(const DevRef& R, const AdvArgs& A, cudaStream_t st) {
  if (A.n_elem <= 0) return cudaSuccess;
  const size_t s1 = adv_trace_smem_doubles<DIM, N>() * sizeof(double), s2 = adv_rhs_smem_doubles<DIM, N>() * sizeof(double);
  static int dev_done[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!dev_done[dev]) {  // the >48 KB opt-in is per device
    if ((e = cudaFuncSetAttribute(adv_trace_kernel<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s1)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(adv_rhs_kernel<DIM, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s2)) != cudaSuccess) return e;
    dev_done[dev] = 1;
  }
  adv_trace_kernel<DIM, N><<<(unsigned)A.n_elem, 128, s1, st>>>(R, A);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  adv_rhs_kernel<DIM, N><<<(unsigned)A.n_elem, 128, s2, st>>>(R, A);
  return cudaGetLastError();
}

template <int N>
static cudaError_t upload_psi_adv(const double* p1, const double* p2, const double* p3) {
  PsiC<N> h;
  for (int k = 0; k < N * N; ++k) h.p1[k] = p1[k];
  for (int k = 0; k < N * N * N; ++k) {
    h.p2[k] = p2[k];
    h.p3[k] = p3[k];
  }
  return cudaMemcpyToSymbol(c_psi<N>, &h, sizeof(h));
}
#define ES_N_CASES(F, ...) \
  switch (n) {           \
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
cudaError_t upload_psi_adv_3d(int n, const double* p1, const double* p2, const double* p3) {
  ES_N_CASES(upload_psi_adv, p1, p2, p3)
}

cudaError_t launch_adv_3d(int n, const DevRef& R, const AdvArgs& A, cudaStream_t st) {
  switch (n) {
    case 2: return do_adv<3, 2>(R, A, st);
    case 3: return do_adv<3, 3>(R, A, st);
    case 4: return do_adv<3, 4>(R, A, st);
    case 5: return do_adv<3, 5>(R, A, st);
    case 6: return do_adv<3, 6>(R, A, st);
    case 7: return do_adv<3, 7>(R, A, st);
    case 8: return do_adv<3, 8>(R, A, st);
    case 9: return do_adv<3, 9>(R, A, st);  
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace esb
