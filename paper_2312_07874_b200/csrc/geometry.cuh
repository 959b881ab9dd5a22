// geometry.cuh -- setup / utility kernel interfaces (product code)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace esb {

struct GeoArgs {
  int dim, Npg, Ncl, Nq, NF, Nqf;
  int gv_stride;        // doubles per element in geo_vol (even: 16-byte aligned element blocks)
  const double* xmap;   // [ne][Npg][dim] mapping-node positions
  // reference matrices as double-double pairs (hi, lo) built in long double (R25)
  const double *LmapV, *DmapV, *DmapF, *DmapM, *LmapC, *DmapC, *DcurlV, *DcurlF;
  const double *LmapV_lo, *DmapV_lo, *DmapF_lo, *DmapM_lo, *LmapC_lo, *DmapC_lo, *DcurlV_lo, *DcurlF_lo;
  const double* Wvol;   // [Nq]
  const double* nhat;   // [Nf][3]
  const double* shift;  // [ne][dim] local-coordinate origin added back to xq (R25)
  double* geo_vol;      // [ne][gv_stride]: [dim*dim+2][Nq] then padding
  double* geo_face;     // [ne][Nf][dim][Nqf]
  double* xq;           // [ne][Nq][dim]
  double* jt_out;       // optional [ne][Nq]
  int* bad;
};

struct FaceCheckArgs {
  int dim, n, Nqf;
  int64_t nloc;
  const double* geo_face;
  const double* Bf;
  const int64_t* face_slot;
  const int* face_reflect;
  unsigned long long* max_mismatch;
};

cudaError_t launch_geometry(const GeoArgs& g, int64_t ne, cudaStream_t st);
cudaError_t launch_face_check(const FaceCheckArgs& a, cudaStream_t st);
cudaError_t launch_pack(const double* trace, const int64_t* slots, int64_t nsend, int per_face, double* buf,
                        cudaStream_t st);
// evaluation at arbitrary reference points (es_eval_points): u = sum_k u~_k psi_k(xi) per variable,
// x = sum_i l_i(xi) X_i, jac = det(sum_i grad l_i(xi) X_i^T) over the element's mapping nodes X
struct EvalPtsArgs {
  int dim, NC, Np, Npg, npts;
  int64_t ne;
  const double* um;    // [ne][NC][Np]
  const double* xmap;  // [ne][Npg][dim] mapping-node positions
  const double* pkd;   // [npts][Np]
  const double* lmap;  // [npts][Npg]
  const double* dmap;  // [dim][npts][Npg]
  double* u;           // [ne][npts][NC]
  double* x;           // optional [ne][npts][dim]
  double* jac;         // optional [ne][npts]
};
cudaError_t launch_eval_points(const EvalPtsArgs& a, cudaStream_t st);

// modal (compressed) metric storage, setup: g~_lm = V^T W G_lm per element
// (exact: the metric terms have degree <= p, R33); one thread per (element, lm, mode)
struct MetricModalArgs {
  int dim, n, Nq, Np, gv_stride, gm_stride;
  int64_t ne;
  const double* geo_vol;                   // [ne][gv_stride]: G rows [NG][Nq] first
  const double *psi1, *psi2, *psi3, *Wvol;  // PKD principal functions [a1][a], [a1][a2][b], [s][a3][c]; weights
  const int *mode_pr, *pair_a1, *pair_a2, *pair_off;
  double* gmod;                            // [ne][gm_stride]: [NG][Np] (+ pad)
};
cudaError_t launch_metric_modal(const MetricModalArgs& a, cudaStream_t st);
cudaError_t launch_reduce_parts(const double* part, int64_t ne, int w, double* out, cudaStream_t st);

// explicit Runge-Kutta combinations over the modal state (HBM-bound streams)
struct RkComb {
  const double* k[16];
  double c[16];  // coefficients of k_j (already multiplied by dt)
  int nk;
};
// out = y0 + sum_j c_j k_j
cudaError_t launch_rk_comb(const double* y0, const RkComb& kc, double* out, int64_t n, cudaStream_t st);
// per-block partial sums of (e_i / (atol + rtol max(|y0_i|, |y1_i|)))^2, e = sum_j c_j k_j, over a
// fixed grid of RK_ERR_BLOCKS blocks (deterministic order) -> part[RK_ERR_BLOCKS]
constexpr int RK_ERR_BLOCKS = 1184;
cudaError_t launch_rk_err(const double* y0, const double* y1, const RkComb& ec, double rtol, double atol,
                          int64_t n, double* part, cudaStream_t st);

}  // namespace esb
