// kernels_3d.cu -- tetrahedron instantiations (q = p = N-1 in [1, 8]) of the kernels in kernels.cuh
#include "kernels.cuh"
#include "rhs2.cuh"

namespace esb {
#include "launch.inc"

#define ES_CASES(F, ...) \
  switch (n) {           \
    case 2: return F<3, 2>(__VA_ARGS__);  \
    case 3: return F<3, 3>(__VA_ARGS__);  \
    case 4: return F<3, 4>(__VA_ARGS__);  \
    case 5: return F<3, 5>(__VA_ARGS__);  \
    case 6: return F<3, 6>(__VA_ARGS__);  \
    case 7: return F<3, 7>(__VA_ARGS__);  \
    case 8: return F<3, 8>(__VA_ARGS__);  \
    case 9: return F<3, 9>(__VA_ARGS__);  \
    default: return cudaErrorInvalidValue; \
  }

// this unit's copy of the constant-memory PKD tables (the 3D psi1 steps of the transforms)
template <int N>
static cudaError_t upload_psi_k1(const double* p1, const double* p2, const double* p3) {
  PsiC<N> h;
  for (int k = 0; k < N * N; ++k) h.p1[k] = p1[k];
  for (int k = 0; k < N * N * N; ++k) {
    h.p2[k] = p2[k];
    h.p3[k] = p3[k];
  }
  return cudaMemcpyToSymbol(c_psi<N>, &h, sizeof(h));
}
#define ES_N_CASES(F, ...)             \
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
cudaError_t upload_psi_3d_k1(int n, const double* p1, const double* p2, const double* p3) {
  ES_N_CASES(upload_psi_k1, p1, p2, p3)
}

cudaError_t launch_project_3d(int n, const DevRef& R, const ProjArgs& A, cudaStream_t st) { ES_CASES(do_project, R, A, st) }
cudaError_t launch_rhs_3d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st) { ES_CASES(do_rhs, R, A, st) }
cudaError_t launch_projnodal_3d(int n, const DevRef& R, int64_t ne, const double* un, double* um, cudaStream_t st) {
  ES_CASES(do_projnodal, R, ne, un, um, st)
}
cudaError_t launch_evalnodal_3d(int n, const DevRef& R, int64_t ne, const double* um, double* un, cudaStream_t st) {
  ES_CASES(do_evalnodal, R, ne, um, un, st)
}
}  // namespace esb
