// advect.cuh -- the linear-advection workload: du/dt + div(a u) = 0 with constant a
// in the skew-symmetric weak form of P:431-436 [eq:rhs_skew] (energy stable on curved meshes), or the
// conservative form P:425-426 [eq:rhs_cons]:
//   r = 1/2 sum_l ( Q^(l)T c_l u - c_l Q^(l) u ) - sum_z R^(z)T B J_f ( f* - 1/2 (a.n) R^(z) u ),
//   c_l = sum_m G_lm a_m at the volume nodes, f* = (a.n)(u- + u+)/2 [- |a.n| (u+ - u-)/2 upwind],
// then d u~/dt = V^T W/J~ V (V^T r) and the RK4 stage update.  Product code.
//
// Q^(l) restricted to an eta_k line is coefficient(line) x X with the unskewed 1D matrices X (Q1, A1..A4,
// tables.cpp; pinned against the oracle's dense Q in tests/test_host_tables.py), so the volume term is a
// line-wise operator application: node i of a k-line gathers its N line partners.  One CTA per element
// (a scalar equation: little work per element), tables staged in shared memory.
#pragma once
#include "kernels.cuh"

namespace esb {

struct AdvArgs {
  int64_t n_elem;
  const double* u;          // [ne][Np] modal stage input
  double* unod;             // [ne][Nq] nodal u (written by the trace kernel)
  double* trace;            // [ne][Nf][Nqf] u at the facet nodes
  const double* geo_vol;    // [ne][GVS]: G_lm rows, W J~, W / J~
  const double* geo_face;   // [ne][Nf][DIM][Nqf] J n
  const int64_t* face_slot;
  const int* face_reflect;
  const double* X;          // [5][N][N] unskewed line matrices fQ1, fA1, fA2, fA3, fA4
  double a[3];              // advection velocity
  int flux_mode;            // 0 central, 1 upwind
  int form;                 // 0 skew-symmetric [eq:rhs_skew], 1 conservative [eq:rhs_cons]
  int mode;                 // 0 dudt, 1..4 RK4 stage (R17)
  double* out;
  const double* u0;
  double* acc;
  double* ustage;
  double dt;
  double* part;             // optional [ne][2]: sum u_i r_i, sum |u_i r_i|
};

// u = V u~ at the volume nodes and its traces R^(z) u at the facet nodes
template <int DIM, int N>
__global__ void __launch_bounds__(128) adv_trace_kernel(DevRef R, AdvArgs A) {
  using S = Sz<DIM, N>;
  constexpr int Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf;
  extern __shared__ __align__(16) double sa[];
  double* un = sa;                          // [Nq]
  double* t1 = un + ((Nq + 1) & ~1);         // t1_size
  double* t2 = t1 + ((t1_size<DIM, N>() + 1) & ~1);
  double* um = t2 + ((t2_size<DIM, N>() + 1) & ~1);  // [Np]
  double* ps = um + ((Np + 1) & ~1);
  const PsiS T = stage_psi<DIM, N>(R, ps);
  const int64_t e = blockIdx.x;
  for (int k = threadIdx.x; k < Np; k += blockDim.x) um[k] = A.u[e * Np + k];
  __syncthreads();
  modal_to_nodal<DIM, N, 1>(T, um, un, t1, t2);
  for (int i = threadIdx.x; i < Nq; i += blockDim.x) A.unod[e * Nq + i] = un[i];
  // traces along lines (facet 4: eta3 first, then eta2), as in K1
  for (int fz = threadIdx.x; fz < NF; fz += blockDim.x) {
    const int z = fz / Nqf, f = fz - z * Nqf;
    double s = 0.0;
    if constexpr (DIM == 2) {
      if (z == 0)
        for (int b = 0; b < N; ++b) s = fma(R.lL[b], un[f + N * b], s);
      else
        for (int a = 0; a < N; ++a) s = fma(z == 1 ? R.lR[a] : R.lL[a], un[a + N * f], s);
    } else {
      const int f1 = f % N, f2 = f / N;
      if (z == 0) {
        for (int b = 0; b < N; ++b) s = fma(R.lL[b], un[f1 + N * b + N * N * f2], s);
      } else if (z < 3) {
        for (int a = 0; a < N; ++a) s = fma(z == 1 ? R.lR[a] : R.lL[a], un[a + N * f1 + N * N * f2], s);
      } else {  // facet 4 (eta3 = -1): node (a = f1, eta3_j = f2): sum_b lint4[j][b] sum_c l3(c) u[a][b][c]
        for (int b = 0; b < N; ++b) {
          double y = 0.0;
          for (int c = 0; c < N; ++c) y = fma(R.l3L[c], un[f1 + N * b + N * N * c], y);
          s = fma(R.lint4[f2 * N + b], y, s);
        }
      }
    }
    A.trace[e * NF + fz] = s;
  }
}

template <int DIM, int N>
__host__ __device__ constexpr size_t adv_trace_smem_doubles() {
  using S = Sz<DIM, N>;
  return ((S::Nq + 1) & ~1) + ((t1_size<DIM, N>() + 1) & ~1) + ((t2_size<DIM, N>() + 1) & ~1) + ((S::Np + 1) & ~1) +
         psi_smem_doubles<DIM, N>();
}

// volume (skew-symmetric or conservative) and surface terms, lifting, weight-adjusted inverse, epilogue
template <int DIM, int N>
__global__ void __launch_bounds__(128) adv_rhs_kernel(DevRef R, AdvArgs A) {
  using S = Sz<DIM, N>;
  constexpr int Nq = S::Nq, Np = S::Np, NF = S::NF, Nqf = S::Nqf, Nf = S::Nf, GVS = S::GVS;
  extern __shared__ __align__(16) double sa[];
  double* un = sa;                                // [Nq] nodal u
  double* cl = un + ((Nq + 1) & ~1);               // [DIM][Nq] c_l = sum_m G_lm a_m
  double* r = cl + ((DIM * Nq + 1) & ~1);          // [Nq] residual
  double* fs = r + ((Nq + 1) & ~1);                // [NF] B J_f (f* - ...)
  double* t1 = fs + ((NF + 1) & ~1);
  double* t2 = t1 + ((t1_size<DIM, N>() + 1) & ~1);
  double* y = t2 + ((t2_size<DIM, N>() + 1) & ~1);  // [Nq]
  double* um = y + ((Nq + 1) & ~1);                // [Np]
  double* X = um + ((Np + 1) & ~1);                // [5][N][N]
  double* ps = X + ((5 * N * N + 1) & ~1);  // 16-byte aligned psi rows
  const PsiS T = stage_psi<DIM, N>(R, ps);
  const int64_t e = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const double* gv = A.geo_vol + (size_t)e * GVS;
  for (int k = tid; k < 5 * N * N; k += nt) X[k] = A.X[k];
  for (int i = tid; i < Nq; i += nt) {
    un[i] = A.unod[e * Nq + i];
    for (int l = 0; l < DIM; ++l) {
      double t = 0.0;
      for (int m = 0; m < DIM; ++m) t = fma(gv[(l * DIM + m) * Nq + i], A.a[m], t);
      cl[l * Nq + i] = t;
    }
  }
  // surface: s_f = B_f J_f (f* - 1/2 (a.n) u-)  (skew) or B_f J_f f* (conservative), own normal
  for (int fz = tid; fz < NF; fz += nt) {
    const int z = fz / Nqf, f = fz - z * Nqf;
    const int64_t slot = A.face_slot[e * Nf + z];
    const int rf = A.face_reflect[e * Nf + z];
    const int fo = DIM == 2 ? (rf ? N - 1 - f : f) : (rf ? (N - 1 - f % N) + N * (f / N) : f);
    const double um_ = A.trace[e * NF + fz], up = A.trace[slot * Nqf + fo];
    double Jf = 0.0, an = 0.0, Jn[3];
    for (int m = 0; m < DIM; ++m) {
      Jn[m] = A.geo_face[((size_t)(e * Nf + z) * DIM + m) * Nqf + f];
      Jf += Jn[m] * Jn[m];
    }
    Jf = sqrt(Jf);
    for (int m = 0; m < DIM; ++m) an += A.a[m] * Jn[m] / Jf;
    double fst = an * 0.5 * (um_ + up);
    if (A.flux_mode == 1) fst -= 0.5 * fabs(an) * (up - um_);
    fs[fz] = __ldg(&R.Bf[fz]) * Jf * (A.form == 0 ? fst - 0.5 * an * um_ : fst);
  }
  __syncthreads();
  // volume: node i gathers its line partners j: Q^(l)_ij = coef X[pos_i][pos_j] on the line
  for (int i = tid; i < Nq; i += nt) {
    const int ca = i % N, cb = (i / N) % N, cc = DIM == 3 ? i / (N * N) : 0;
    double acc = 0.0;
    for (int k = 0; k < DIM; ++k) {
      const int pos = k == 0 ? ca : (k == 1 ? cb : cc);
      const int stride = k == 0 ? 1 : (k == 1 ? N : N * N);
      // (operator l, matrix index, coefficient) contributions of this line direction
      int lop[3], xm[3], nop = 0;
      double co = 0.0;
      if constexpr (DIM == 2) {
        if (k == 0) {
          co = R.w[cb];
          lop[0] = 0, xm[0] = 0, lop[1] = 1, xm[1] = 1, nop = 2;
        } else {
          co = R.w[ca];
          lop[0] = 1, xm[0] = 2, nop = 1;
        }
      } else {
        if (k == 0) {
          co = 0.5 * R.w[cb] * R.w3[cc];
          lop[0] = 0, xm[0] = 0, lop[1] = 1, xm[1] = 1, lop[2] = 2, xm[2] = 1, nop = 3;
        } else if (k == 1) {
          co = 0.5 * R.w[ca] * R.w3[cc];
          lop[0] = 1, xm[0] = 2, lop[1] = 2, xm[1] = 3, nop = 2;
        } else {
          co = 0.125 * R.w[ca] * R.w[cb] * (1.0 - R.eta[cb]);
          lop[0] = 2, xm[0] = 4, nop = 1;
        }
      }
      for (int q = 0; q < nop; ++q) {
        const double* Xm = X + xm[q] * N * N;
        const double* c = cl + lop[q] * Nq;
        double t = 0.0;
        for (int b = 0; b < N; ++b) {
          const int j = i + (b - pos) * stride;
          const double qt = Xm[b * N + pos] * c[j] * un[j];  // (Q^T (c u))_i
          t += A.form == 0 ? 0.5 * (qt - c[i] * Xm[pos * N + b] * un[j]) : qt;
        }
        acc = fma(co, t, acc);
      }
    }
    // lifting r -= R^T s along the lines (facet 4 through the eta3 and eta2 extrapolations)
    double lift;
    if constexpr (DIM == 2) {
      lift = R.lL[cb] * fs[0 * Nqf + ca] + R.lR[ca] * fs[1 * Nqf + cb] + R.lL[ca] * fs[2 * Nqf + cb];
    } else {
      double f4 = 0.0;
      for (int jf = 0; jf < N; ++jf) f4 = fma(R.lint4[jf * N + cb], fs[3 * Nqf + ca + N * jf], f4);
      lift = R.lL[cb] * fs[0 * Nqf + ca + N * cc] + R.lR[ca] * fs[1 * Nqf + cb + N * cc] +
             R.lL[ca] * fs[2 * Nqf + cb + N * cc] + R.l3L[cc] * f4;
    }
    r[i] = acc - lift;
  }
  __syncthreads();
  if (A.part) {  // energy rate sum u^T r = d/dt sum u~^T M~ u~ / 2 and its scale (deterministic)
    double s0 = 0.0, s1 = 0.0;
    for (int i = tid; i < Nq; i += nt) {
      const double t = un[i] * r[i];
      s0 += t;
      s1 += fabs(t);
    }
    __shared__ double red[2][32];
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_down_sync(0xffffffffu, s0, o);
      s1 += __shfl_down_sync(0xffffffffu, s1, o);
    }
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = s0;
      red[1][tid >> 5] = s1;
    }
    __syncthreads();
    if (tid == 0) {
      double a0 = 0.0, a1 = 0.0;
      for (int w = 0; w < nt / 32; ++w) {
        a0 += red[0][w];
        a1 += red[1][w];
      }
      A.part[e * 2] = a0;
      A.part[e * 2 + 1] = a1;
    }
  }
  // d u~/dt = V^T W/J~ V (V^T r)
  nodal_to_modal<DIM, N, 1>(T, r, um, t1, t2);
  modal_to_nodal<DIM, N, 1>(T, um, y, t1, t2);
  nodal_to_modal<DIM, N, 1>(T, y, um, t1, t2, gv + (S::NG + 1) * Nq);
  const size_t base = (size_t)e * Np;
  const double dt = A.dt;
  for (int k = tid; k < Np; k += nt) {
    const double du = um[k];
    switch (A.mode) {
      case 0:
        A.out[base + k] = du;
        break;
      case 1:
        A.acc[base + k] = A.u0[base + k] + (dt / 6.0) * du;
        A.ustage[base + k] = A.u0[base + k] + (0.5 * dt) * du;
        break;
      case 2:
        A.acc[base + k] += (dt / 3.0) * du;
        A.ustage[base + k] = A.u0[base + k] + (0.5 * dt) * du;
        break;
      case 3:
        A.acc[base + k] += (dt / 3.0) * du;
        A.ustage[base + k] = A.u0[base + k] + dt * du;
        break;
      case 4:
        A.out[base + k] = A.acc[base + k] + (dt / 6.0) * du;
        break;
    }
  }
}

template <int DIM, int N>
__host__ __device__ constexpr size_t adv_rhs_smem_doubles() {
  using S = Sz<DIM, N>;
  return ((S::Nq + 1) & ~1) * 3 + ((DIM * S::Nq + 1) & ~1) + ((S::NF + 1) & ~1) + ((t1_size<DIM, N>() + 1) & ~1) +
         ((t2_size<DIM, N>() + 1) & ~1) + ((S::Np + 1) & ~1) + ((5 * N * N + 1) & ~1) + psi_smem_doubles<DIM, N>();
}

}  // namespace esb
