// kernels_2d.cu -- triangle instantiations (q = p = N-1 in [1, 10]) of the kernels in kernels.cuh
#include "kernels.cuh"
#include "rhs2.cuh"

namespace esb {
#include "launch.inc"

#define ES_CASES(F, ...) \
  switch (n) {           \
    case 2: return F<2, 2>(__VA_ARGS__);  \
    case 3: return F<2, 3>(__VA_ARGS__);  \
    case 4: return F<2, 4>(__VA_ARGS__);  \
    case 5: return F<2, 5>(__VA_ARGS__);  \
    case 6: return F<2, 6>(__VA_ARGS__);  \
    case 7: return F<2, 7>(__VA_ARGS__);  \
    case 8: return F<2, 8>(__VA_ARGS__);  \
    case 9: return F<2, 9>(__VA_ARGS__);  \
    case 10: return F<2, 10>(__VA_ARGS__); \
    case 11: return F<2, 11>(__VA_ARGS__); \
    default: return cudaErrorInvalidValue; \
  }

cudaError_t launch_project_2d(int n, const DevRef& R, const ProjArgs& A, cudaStream_t st) { ES_CASES(do_project, R, A, st) }
cudaError_t launch_rhs_2d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st) { ES_CASES(do_rhs, R, A, st) }
cudaError_t launch_projnodal_2d(int n, const DevRef& R, int64_t ne, const double* un, double* um, cudaStream_t st) {
  ES_CASES(do_projnodal, R, ne, un, um, st)
}
cudaError_t launch_evalnodal_2d(int n, const DevRef& R, int64_t ne, const double* um, double* un, cudaStream_t st) {
  ES_CASES(do_evalnodal, R, ne, um, un, st)
}
}  // namespace esb
