// kernels_2d_cnt.cu -- counting instantiations of the 2D flux kernel (es_count_fluxes): the production
// line-wise kernel and the Eq. num_fluxes ablation with per-element flux-evaluation counters
#define ES_COUNT_TU
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

cudaError_t launch_rhs_count_2d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st) { ES_CASES(do_rhs_count, R, A, st) }
}  // namespace esb
