// adv_2d.cu -- instantiations of the linear-advection kernels (advect.cuh) for triangles
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

cudaError_t launch_adv_2d(int n, const DevRef& R, const AdvArgs& A, cudaStream_t st) {
  switch (n) {
    case 2: return do_adv<2, 2>(R, A, st);
    case 3: return do_adv<2, 3>(R, A, st);
    case 4: return do_adv<2, 4>(R, A, st);
    case 5: return do_adv<2, 5>(R, A, st);
    case 6: return do_adv<2, 6>(R, A, st);
    case 7: return do_adv<2, 7>(R, A, st);
    case 8: return do_adv<2, 8>(R, A, st);
    case 9: return do_adv<2, 9>(R, A, st);
    case 10: return do_adv<2, 10>(R, A, st);
    case 11: return do_adv<2, 11>(R, A, st);  
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace esb
