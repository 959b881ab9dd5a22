// oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// A plain, dense, step-by-step CPU implementation of the entropy-stable modal DSEM right-hand side
// of Montoya & Zingg (arXiv 2312.07874), written from PAPER.md.  Every function cites the passage
// it follows (P:<line> [label]).  It deliberately uses dense matrices and the paper's formulas as
// printed (with the corrections listed as readings R1..R24 in DESIGN.md section 3); there is no
// blocking, fusion or reordering beyond what the paper states.  It shares no code with the CUDA
// product path.  Build: g++ -O2 -ffp-contract=off -fopenmp -shared -fPIC.
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

using std::vector;

namespace {

const double PI = 3.14159265358979323846;

// ------------------------------------------------------------------------------------------------
// 1D: normalised Jacobi polynomials, computed with the three-term recurrence for the
// orthonormal family (Hesthaven & Warburton App. A, cited at P:144).
// ------------------------------------------------------------------------------------------------
template <class T>
struct JacobiRecT {
  // P_{i+1} = ((x - bn[i]) P_i - ao[i] P_{i-1}) / an[i]
  T p0, c1;
  vector<T> an, bn, ao;
};
using JacobiRec = JacobiRecT<double>;

template <class T>
JacobiRecT<T> jacobi_recT(int nmax, T a, T b) {
  JacobiRecT<T> r;
  r.p0 = std::sqrt(std::pow((T)2.0, -a - b - (T)1.0) * std::tgamma(a + b + (T)2.0) /
                   (std::tgamma(a + (T)1.0) * std::tgamma(b + (T)1.0)));
  r.c1 = std::sqrt((a + b + (T)3.0) / ((a + (T)1.0) * (b + (T)1.0)));
  T aold = (T)2.0 / ((T)2.0 + a + b) * std::sqrt((a + (T)1.0) * (b + (T)1.0) / (a + b + (T)3.0));
  r.an.assign(nmax + 1, (T)0.0);
  r.bn.assign(nmax + 1, (T)0.0);
  r.ao.assign(nmax + 1, (T)0.0);
  for (int i = 1; i <= nmax; ++i) {
    T h1 = (T)2.0 * i + a + b;
    T anew = (T)2.0 / (h1 + (T)2.0) *
             std::sqrt(((T)i + 1) * ((T)i + 1 + a + b) * ((T)i + 1 + a) * ((T)i + 1 + b) /
                       ((h1 + (T)1.0) * (h1 + (T)3.0)));
    T bnew = -(a * a - b * b) / (h1 * (h1 + (T)2.0));
    r.an[i] = anew;
    r.bn[i] = bnew;
    r.ao[i] = aold;
    aold = anew;
  }
  return r;
}
JacobiRec jacobi_rec(int nmax, double a, double b) { return jacobi_recT<double>(nmax, a, b); }

template <class T>
T jacobi_val(int n, T a, T b, T x) {
  JacobiRecT<T> r = jacobi_recT<T>(n, a, b);
  T pm = r.p0;
  if (n == 0) return pm;
  T pc = r.p0 * ((a + b + (T)2) * x / (T)2 + (a - b) / (T)2) * r.c1;
  for (int i = 1; i < n; ++i) {
    T pn = ((x - r.bn[i]) * pc - r.ao[i] * pm) / r.an[i];
    pm = pc;
    pc = pn;
  }
  return pc;
}
template <class T>
T jacobi_der(int n, T a, T b, T x) {
  if (n == 0) return 0;
  return std::sqrt((T)n * ((T)n + a + b + (T)1)) * jacobi_val<T>(n - 1, a + (T)1, b + (T)1, x);
}

double jacobi(int n, double a, double b, double x) {
  JacobiRec r = jacobi_rec(n, a, b);
  double pm = r.p0;
  if (n == 0) return pm;
  double pc = r.p0 * ((a + b + 2.0) * x / 2.0 + (a - b) / 2.0) * r.c1;
  for (int i = 1; i < n; ++i) {
    double pn = ((x - r.bn[i]) * pc - r.ao[i] * pm) / r.an[i];
    pm = pc;
    pc = pn;
  }
  return pc;
}

// d/dx P_n^(a,b) = sqrt(n (n+a+b+1)) P_{n-1}^(a+1,b+1)  (normalised family)
double jacobi_deriv(int n, double a, double b, double x) {
  if (n == 0) return 0.0;
  return std::sqrt(n * (n + a + b + 1.0)) * jacobi(n - 1, a + 1.0, b + 1.0, x);
}

// Gauss rule ("Gauss: P_{q+1}^(a,b)(eta) = 0"): Newton iteration with polynomial deflation
// (Karniadakis & Sherwin App. B, cited at P:160); weights from the Christoffel numbers of the
// orthonormal family, w_i = 1 / sum_{k<=q} P_k(x_i)^2, equal to int l_i (1-x)^a (1+x)^b.
// All reference tables are computed in long double and rounded once to FP64 (reading R26).
typedef long double LD;
template <class T>
void gauss_jacobiT(int q, T a, T b, vector<T>& x, vector<T>& w) {
  int N = q + 1;
  x.assign(N, (T)0);
  w.assign(N, (T)0);
  for (int k = 0; k < N; ++k) {
    T r = -std::cos(((T)2 * k + (T)1) * (T)PI / ((T)2 * N));
    if (k > 0) r = (r + x[k - 1]) / (T)2;
    for (int it = 0; it < 200; ++it) {
      T s = 0;
      for (int j = 0; j < k; ++j) s += (T)1 / (r - x[j]);
      T P = jacobi_val<T>(N, a, b, r);
      T dP = jacobi_der<T>(N, a, b, r);
      T delta = -P / (dP - s * P);
      r += delta;
      if (std::fabs(delta) < (T)1e-19 * ((T)1 + std::fabs(r))) break;
    }
    x[k] = r;
  }
  std::sort(x.begin(), x.end());
  for (int i = 0; i < N; ++i) {
    T s = 0;
    for (int k = 0; k < N; ++k) {
      T pk = jacobi_val<T>(k, a, b, x[i]);
      s += pk * pk;
    }
    w[i] = (T)1 / s;
  }
}
void gauss_jacobi(int q, double a, double b, vector<double>& x, vector<double>& w) {
  vector<LD> xl, wl;
  gauss_jacobiT<LD>(q, a, b, xl, wl);
  x.assign(xl.begin(), xl.end());
  w.assign(wl.begin(), wl.end());
}

// Lagrange polynomials (P:153-155 [eq:lagrange]) and their derivatives, by the product formula.
template <class T>
T lagrange(const vector<T>& nd, int j, T x) {
  T v = 1;
  for (size_t k = 0; k < nd.size(); ++k)
    if ((int)k != j) v *= (x - nd[k]) / (nd[j] - nd[k]);
  return v;
}
template <class T>
T lagrange_deriv(const vector<T>& nd, int j, T x) {
  T s = 0;
  for (size_t k = 0; k < nd.size(); ++k) {
    if ((int)k == j) continue;
    T t = (T)1 / (nd[j] - nd[k]);
    for (size_t m = 0; m < nd.size(); ++m)
      if ((int)m != j && m != k) t *= (x - nd[m]) / (nd[j] - nd[m]);
    s += t;
  }
  return s;
}

// ------------------------------------------------------------------------------------------------
// Reference element with dense operators, and the PKD basis.
// ------------------------------------------------------------------------------------------------
struct Ref {
  int d, q, n, Nq, Nf, Nqf, p, Np;
  vector<double> eta1, w1, eta3, w3;  // LG (0,0) and GJ (1,0) rules (tet uses eta3)
  vector<double> eta;                 // [Nq][d] collapsed coordinates of the volume nodes
  vector<double> xi;                  // [Nq][d]
  vector<double> W;                   // [Nq]
  vector<double> xif;                 // [Nf][Nqf][d]
  vector<double> B;                   // [Nf][Nqf]
  vector<double> nhat;                // [Nf][d]
  vector<double> D, Q, E, S;          // [d][Nq][Nq]
  vector<double> R;                   // [Nf][Nqf][Nq]
  vector<int> alpha;                  // [Np][d]
  vector<double> V;                   // [Nq][Np]
  vector<int> line_dir;               // not used by the oracle loops; kept for clarity
};

// Tetrahedral collapsed map with the corrected first component (R1):
// xi1 = 1/4 (1+eta1)(1-eta2)(1-eta3) - 1   (P:263 prints (1-eta2)(1-eta2)).
template <class T>
void chi(int d, const T* e, T* x) {
  if (d == 2) {  // P:183 [eq:tri_mapping]
    x[0] = (T)0.5 * ((T)1 + e[0]) * ((T)1 - e[1]) - (T)1;
    x[1] = e[1];
  } else {  // P:263 [eq:tet_mapping], R1
    x[0] = (T)0.25 * ((T)1 + e[0]) * ((T)1 - e[1]) * ((T)1 - e[2]) - (T)1;
    x[1] = (T)0.5 * ((T)1 + e[1]) * ((T)1 - e[2]) - (T)1;
    x[2] = e[2];
  }
}

// Multi-index order pi (R9): alpha1-major nested.
vector<int> multi_indices(int d, int p) {
  vector<int> al;
  for (int a1 = 0; a1 <= p; ++a1)
    for (int a2 = 0; a2 <= p - a1; ++a2) {
      if (d == 2) {
        al.push_back(a1);
        al.push_back(a2);
      } else {
        for (int a3 = 0; a3 <= p - a1 - a2; ++a3) {
          al.push_back(a1);
          al.push_back(a2);
          al.push_back(a3);
        }
      }
    }
  return al;
}

// PKD basis function from the principal functions (P:378-389 [eq:principal_functions,
// eq:modal_basis_2d/3d]), evaluated at collapsed coordinates eta.
template <class T>
T pkd_eta(int d, const int* al, const T* e) {
  T v = std::sqrt((T)2) * jacobi_val<T>(al[0], 0, 0, e[0]);
  v *= std::pow((T)1 - e[1], (T)al[0]) * jacobi_val<T>(al[1], (T)2 * al[0] + (T)1, 0, e[1]);
  if (d == 3)
    v *= (T)2 * std::pow((T)1 - e[2], (T)(al[0] + al[1])) *
         jacobi_val<T>(al[2], (T)2 * al[0] + (T)2 * al[1] + (T)2, 0, e[2]);
  return v;
}

// The same PKD functions written in Cartesian (homogenised) form so that values and gradients are
// defined everywhere on the closed simplex, including the collapsed vertex:
//   t^i P_i(s/t) obeys the homogenised recurrence H_{i+1} = ((s - b_i t) H_i - a_i t^2 H_{i-1})/a'_i.
// tri:  phi = sqrt2 2^a1 H_a1^(0,0)(s,t) P_a2^(2a1+1,0)(xi2),  t=(1-xi2)/2, s=(1+xi1)-t
// tet:  phi = 2 sqrt2 4^a1 2^a2 H_a1^(0,0)(s1,t1) H_a2^(2a1+1,0)(s2,t2) P_a3^(2a1+2a2+2,0)(xi3),
//       t1=(-xi2-xi3)/2, s1=(1+xi1)-t1, t2=(1-xi3)/2, s2=(1+xi2)-t2.
template <class T>
void homog(int n, T a, T b, T s, const T* ds, T t, const T* dt, int d, T& H, T* dH) {
  JacobiRecT<T> r = jacobi_recT<T>(n + 1, a, b);
  T Hm = r.p0, dHm[3] = {0, 0, 0};
  if (n == 0) {
    H = Hm;
    for (int k = 0; k < d; ++k) dH[k] = 0.0;
    return;
  }
  T c = r.p0 * r.c1;
  T Hc = c * ((a + b + (T)2.0) * s / (T)2.0 + (a - b) * t / (T)2.0);
  T dHc[3];
  for (int k = 0; k < d; ++k) dHc[k] = c * ((a + b + (T)2.0) * ds[k] / (T)2.0 + (a - b) * dt[k] / (T)2.0);
  for (int i = 1; i < n; ++i) {
    T Hn = ((s - r.bn[i] * t) * Hc - r.ao[i] * t * t * Hm) / r.an[i];
    T dHn[3];
    for (int k = 0; k < d; ++k)
      dHn[k] = ((ds[k] - r.bn[i] * dt[k]) * Hc + (s - r.bn[i] * t) * dHc[k] -
                r.ao[i] * ((T)2.0 * t * dt[k] * Hm + t * t * dHm[k])) /
               r.an[i];
    Hm = Hc;
    Hc = Hn;
    for (int k = 0; k < d; ++k) {
      dHm[k] = dHc[k];
      dHc[k] = dHn[k];
    }
  }
  H = Hc;
  for (int k = 0; k < d; ++k) dH[k] = dHc[k];
}

template <class T>
T jacobiT(int n, T a, T b, T x) {
  T H, dH[1];
  T one = 1.0, zero = 0.0;
  homog<T>(n, a, b, x, &one, one, &zero, 1, H, dH);
  return H;
}
template <class T>
T jacobi_derivT(int n, T a, T b, T x) {
  if (n == 0) return 0.0;
  return std::sqrt((T)n * ((T)n + a + b + (T)1.0)) * jacobiT<T>(n - 1, a + (T)1.0, b + (T)1.0, x);
}

template <class T>
void pkd_cart(int d, const int* al, const T* x, T& v, T* g) {
  if (d == 2) {
    T t = ((T)1.0 - x[1]) / (T)2.0, s = ((T)1.0 + x[0]) - t;
    T dt[2] = {0.0, -0.5}, ds[2] = {1.0, 0.5};
    T H, dH[2];
    homog<T>(al[0], 0, 0, s, ds, t, dt, 2, H, dH);
    T P = jacobiT<T>(al[1], (T)2.0 * al[0] + (T)1.0, 0, x[1]);
    T dP = jacobi_derivT<T>(al[1], (T)2.0 * al[0] + (T)1.0, 0, x[1]);
    T c = std::sqrt((T)2.0) * std::pow((T)2.0, (T)al[0]);
    v = c * H * P;
    g[0] = c * dH[0] * P;
    g[1] = c * (dH[1] * P + H * dP);
  } else {
    T t1 = (-x[1] - x[2]) / (T)2.0, s1 = ((T)1.0 + x[0]) - t1;
    T dt1[3] = {0.0, -0.5, -0.5}, ds1[3] = {1.0, 0.5, 0.5};
    T t2 = ((T)1.0 - x[2]) / (T)2.0, s2 = ((T)1.0 + x[1]) - t2;
    T dt2[3] = {0.0, 0.0, -0.5}, ds2[3] = {0.0, 1.0, 0.5};
    T H1, dH1[3], H2, dH2[3];
    homog<T>(al[0], 0, 0, s1, ds1, t1, dt1, 3, H1, dH1);
    homog<T>(al[1], (T)2.0 * al[0] + (T)1.0, 0, s2, ds2, t2, dt2, 3, H2, dH2);
    T a3 = (T)2.0 * al[0] + (T)2.0 * al[1] + (T)2.0;
    T P = jacobiT<T>(al[2], a3, 0, x[2]);
    T dP = jacobi_derivT<T>(al[2], a3, 0, x[2]);
    T c = (T)2.0 * std::sqrt((T)2.0) * std::pow((T)4.0, (T)al[0]) * std::pow((T)2.0, (T)al[1]);
    v = c * H1 * H2 * P;
    for (int k = 0; k < 3; ++k) g[k] = c * (dH1[k] * H2 * P + H1 * dH2[k] * P);
    g[2] += c * H1 * H2 * dP;
  }
}

Ref build_ref(int d, int q, int p) {
  // every table is evaluated in long double and rounded once to FP64 (reading R26)
  Ref r;
  r.d = d;
  r.q = q;
  r.n = q + 1;
  int n = r.n;
  r.Nq = (d == 2) ? n * n : n * n * n;
  r.Nf = d + 1;
  r.Nqf = (d == 2) ? n : n * n;
  r.p = p;
  const int Nq = r.Nq, Nqf = r.Nqf, Nf = r.Nf;
  vector<LD> e, w, e3, w3;
  gauss_jacobiT<LD>(q, 0, 0, e, w);
  gauss_jacobiT<LD>(q, 1, 0, e3, w3);
  r.eta1.assign(e.begin(), e.end());
  r.w1.assign(w.begin(), w.end());
  r.eta3.assign(e3.begin(), e3.end());
  r.w3.assign(w3.begin(), w3.end());
  vector<LD> eta((size_t)Nq * d), xi((size_t)Nq * d), W(Nq), xif((size_t)Nf * Nqf * d), B((size_t)Nf * Nqf),
      nhat((size_t)Nf * d);
  auto sg = [&](int a, int b, int c) { return a + n * b + n * n * c; };  // sigma (R9)
  if (d == 2) {
    // P:205 [eq:tri_quadrature]
    for (int b = 0; b < n; ++b)
      for (int a = 0; a < n; ++a) {
        int i = sg(a, b, 0);
        LD et[2] = {e[a], e[b]};
        eta[i * 2] = e[a];
        eta[i * 2 + 1] = e[b];
        chi<LD>(2, et, &xi[i * 2]);
        W[i] = ((LD)1 - e[b]) / (LD)2 * w[a] * w[b];
      }
    // P:208-212 [eq:tri_facet_quadrature_nodes]
    for (int i = 0; i < n; ++i) {
      LD f1[2] = {e[i], -1}, f2[2] = {1, e[i]}, f3[2] = {-1, e[i]};
      chi<LD>(2, f1, &xif[(0 * n + i) * 2]);
      chi<LD>(2, f2, &xif[(1 * n + i) * 2]);
      chi<LD>(2, f3, &xif[(2 * n + i) * 2]);
      B[0 * n + i] = w[i];
      B[1 * n + i] = std::sqrt((LD)2) * w[i];
      B[2 * n + i] = w[i];
    }
    // outward unit normals of the facets P:176-178
    LD r2 = (LD)1 / std::sqrt((LD)2);
    LD nh[6] = {0, -1, r2, r2, -1, 0};
    for (int k = 0; k < 6; ++k) nhat[k] = nh[k];
  } else {
    // P:267 [eq:tet_quadrature]
    for (int c = 0; c < n; ++c)
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          int i = sg(a, b, c);
          LD et[3] = {e[a], e[b], e3[c]};
          for (int k = 0; k < 3; ++k) eta[i * 3 + k] = et[k];
          chi<LD>(3, et, &xi[i * 3]);
          W[i] = ((LD)1 - e[b]) * ((LD)1 - e3[c]) / (LD)8 * w[a] * w[b] * w3[c];
        }
    // P:271-283 [eq:tet_facet_quadrature_nodes, eq:tet_facet_quadrature_weights]
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int f = i + n * j;  // sigma_f (R9)
        LD f1[3] = {e[i], -1, e3[j]}, f2[3] = {1, e[i], e3[j]}, f3[3] = {-1, e[i], e3[j]}, f4[3] = {e[i], e3[j], -1};
        chi<LD>(3, f1, &xif[(0 * Nqf + f) * 3]);
        chi<LD>(3, f2, &xif[(1 * Nqf + f) * 3]);
        chi<LD>(3, f3, &xif[(2 * Nqf + f) * 3]);
        chi<LD>(3, f4, &xif[(3 * Nqf + f) * 3]);
        B[0 * Nqf + f] = w[i] * w3[j] / (LD)2;
        B[1 * Nqf + f] = std::sqrt((LD)3) / (LD)2 * w[i] * w3[j];
        B[2 * Nqf + f] = w[i] * w3[j] / (LD)2;
        B[3 * Nqf + f] = w[i] * w3[j] / (LD)2;
      }
    // outward unit normals of the facets P:257-258
    LD s3 = (LD)1 / std::sqrt((LD)3);
    LD nh[12] = {0, -1, 0, s3, s3, s3, -1, 0, 0, 0, 0, -1};
    for (int k = 0; k < 12; ++k) nhat[k] = nh[k];
  }
  // derivative operators P:218-221 [eq:d_2d] and P:286-289 [eq:d_3d] (R2: delta_{a3 b3})
  vector<LD> D((size_t)d * Nq * Nq, (LD)0);
  auto Dm = [&](int m, int i, int j) -> LD& { return D[((size_t)m * Nq + i) * Nq + j]; };
  if (d == 2) {
    for (int b = 0; b < n; ++b)
      for (int a = 0; a < n; ++a)
        for (int bb = 0; bb < n; ++bb)
          for (int aa = 0; aa < n; ++aa) {
            int i = sg(a, b, 0), j = sg(aa, bb, 0);
            LD dl1 = lagrange_deriv<LD>(e, aa, e[a]);
            LD dl2 = lagrange_deriv<LD>(e, bb, e[b]);
            LD d_ab = (b == bb) ? 1 : 0, d_aa = (a == aa) ? 1 : 0;
            Dm(0, i, j) = (LD)2 / ((LD)1 - e[b]) * dl1 * d_ab;
            Dm(1, i, j) = ((LD)1 + e[a]) / ((LD)1 - e[b]) * dl1 * d_ab + d_aa * dl2;
          }
  } else {
    for (int c = 0; c < n; ++c)
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a)
          for (int cc = 0; cc < n; ++cc)
            for (int bb = 0; bb < n; ++bb)
              for (int aa = 0; aa < n; ++aa) {
                int i = sg(a, b, c), j = sg(aa, bb, cc);
                LD d1 = (a == aa) ? 1 : 0, d2 = (b == bb) ? 1 : 0, d3 = (c == cc) ? 1 : 0;
                if (d1 == 0 && d2 == 0) continue;  // no term couples such nodes
                LD dl1 = lagrange_deriv<LD>(e, aa, e[a]);
                LD dl2 = lagrange_deriv<LD>(e, bb, e[b]);
                LD dl3 = lagrange_deriv<LD>(e3, cc, e3[c]);
                LD den = ((LD)1 - e[b]) * ((LD)1 - e3[c]);
                Dm(0, i, j) = (LD)4 / den * dl1 * d2 * d3;
                Dm(1, i, j) = (LD)2 * ((LD)1 + e[a]) / den * dl1 * d2 * d3 + (LD)2 / ((LD)1 - e3[c]) * d1 * dl2 * d3;
                Dm(2, i, j) = (LD)2 * ((LD)1 + e[a]) / den * dl1 * d2 * d3 +
                              ((LD)1 + e[b]) / ((LD)1 - e3[c]) * d1 * dl2 * d3 + d1 * d2 * dl3;
              }
  }
  // extrapolation operators P:223-227 [eq:r_2d] and P:292-297 [eq:r_3d]
  vector<LD> R((size_t)Nf * Nqf * Nq, (LD)0);
  auto Rz = [&](int z, int f, int j) -> LD& { return R[((size_t)z * Nqf + f) * Nq + j]; };
  if (d == 2) {
    for (int i = 0; i < n; ++i)
      for (int bb = 0; bb < n; ++bb)
        for (int aa = 0; aa < n; ++aa) {
          int j = sg(aa, bb, 0);
          Rz(0, i, j) = lagrange<LD>(e, aa, e[i]) * lagrange<LD>(e, bb, -1);
          Rz(1, i, j) = lagrange<LD>(e, aa, 1) * lagrange<LD>(e, bb, e[i]);
          Rz(2, i, j) = lagrange<LD>(e, aa, -1) * lagrange<LD>(e, bb, e[i]);
        }
  } else {
    for (int a2 = 0; a2 < n; ++a2)
      for (int a1 = 0; a1 < n; ++a1)
        for (int cc = 0; cc < n; ++cc)
          for (int bb = 0; bb < n; ++bb)
            for (int aa = 0; aa < n; ++aa) {
              int f = a1 + n * a2, j = sg(aa, bb, cc);
              Rz(0, f, j) = lagrange<LD>(e, aa, e[a1]) * lagrange<LD>(e, bb, -1) * lagrange<LD>(e3, cc, e3[a2]);
              Rz(1, f, j) = lagrange<LD>(e, aa, 1) * lagrange<LD>(e, bb, e[a1]) * lagrange<LD>(e3, cc, e3[a2]);
              Rz(2, f, j) = lagrange<LD>(e, aa, -1) * lagrange<LD>(e, bb, e[a1]) * lagrange<LD>(e3, cc, e3[a2]);
              Rz(3, f, j) = lagrange<LD>(e, aa, e[a1]) * lagrange<LD>(e, bb, e3[a2]) * lagrange<LD>(e3, cc, -1);
            }
  }
  // Q = W D, E = sum_z nhat_m R^T B R (P:131 [eq:e_decomp]), S = Q - E/2
  vector<LD> Q((size_t)d * Nq * Nq, (LD)0), E((size_t)d * Nq * Nq, (LD)0), S((size_t)d * Nq * Nq, (LD)0);
  for (int m = 0; m < d; ++m) {
    for (int i = 0; i < Nq; ++i)
      for (int j = 0; j < Nq; ++j) Q[((size_t)m * Nq + i) * Nq + j] = W[i] * Dm(m, i, j);
    for (int z = 0; z < Nf; ++z) {
      LD nm = nhat[z * d + m];
      if (nm == 0) continue;
      for (int f = 0; f < Nqf; ++f) {
        LD bf = B[z * Nqf + f];
        for (int i = 0; i < Nq; ++i) {
          LD ri = Rz(z, f, i);
          if (ri == 0) continue;
          for (int j = 0; j < Nq; ++j) E[((size_t)m * Nq + i) * Nq + j] += nm * ri * bf * Rz(z, f, j);
        }
      }
    }
    for (size_t k = 0; k < (size_t)Nq * Nq; ++k)
      S[(size_t)m * Nq * Nq + k] = Q[(size_t)m * Nq * Nq + k] - E[(size_t)m * Nq * Nq + k] / (LD)2;
  }
  // generalised Vandermonde V_ij = phi_j(xi_i) (P:372-374 [eq:modal_to_nodal])
  r.alpha = multi_indices(d, p);
  r.Np = (int)r.alpha.size() / d;
  vector<LD> V((size_t)Nq * r.Np);
  for (int i = 0; i < Nq; ++i)
    for (int k = 0; k < r.Np; ++k) V[(size_t)i * r.Np + k] = pkd_eta<LD>(d, &r.alpha[k * d], &eta[i * d]);
  auto rd = [](const vector<LD>& v) { return vector<double>(v.begin(), v.end()); };
  r.eta = rd(eta);
  r.xi = rd(xi);
  r.W = rd(W);
  r.xif = rd(xif);
  r.B = rd(B);
  r.nhat = rd(nhat);
  r.D = rd(D);
  r.Q = rd(Q);
  r.E = rd(E);
  r.S = rd(S);
  r.R = rd(R);
  r.V = rd(V);
  return r;
}

// ------------------------------------------------------------------------------------------------
// Euler physics and SURVEY App. B formulas for the entropy variables.
// ------------------------------------------------------------------------------------------------
struct Prim {
  double rho, v[3], p;
};
Prim prim(int d, double g, const double* U) {
  Prim s;
  s.rho = U[0];
  double ke = 0.0;
  for (int k = 0; k < d; ++k) {
    s.v[k] = U[1 + k] / U[0];
    ke += s.v[k] * U[1 + k];
  }
  s.p = (g - 1.0) * (U[d + 1] - 0.5 * ke);
  return s;
}
// W(U) = grad_U S for S = -rho ln(p/rho^g)/(g-1) (R7):
// W = ((g - s)/(g-1) - beta |v|^2 / 2, beta v, -beta),  s = ln p - g ln rho, beta = rho/p
void entropy_vars(int d, double g, const double* U, double* Wv) {
  Prim s = prim(d, g, U);
  double ent = std::log(s.p) - g * std::log(s.rho);
  double beta = s.rho / s.p;
  double v2 = 0.0;
  for (int k = 0; k < d; ++k) v2 += s.v[k] * s.v[k];
  Wv[0] = (g - ent) / (g - 1.0) - 0.5 * beta * v2;
  for (int k = 0; k < d; ++k) Wv[1 + k] = beta * s.v[k];
  Wv[d + 1] = -beta;
}
// inverse map U(W) (R7): b = -w_last, v = w_mid/b, s = g - (g-1)(w1 + b|v|^2/2),
// rho = (b e^s)^(1/(1-g)), p = rho/b, E = p/(g-1) + rho|v|^2/2
void cons_from_entropy(int d, double g, const double* Wv, double* U) {
  double b = -Wv[d + 1];
  double v[3], v2 = 0.0;
  for (int k = 0; k < d; ++k) {
    v[k] = Wv[1 + k] / b;
    v2 += v[k] * v[k];
  }
  double s = g - (g - 1.0) * (Wv[0] + 0.5 * b * v2);
  double rho = std::pow(b * std::exp(s), 1.0 / (1.0 - g));
  double p = rho / b;
  U[0] = rho;
  for (int k = 0; k < d; ++k) U[1 + k] = rho * v[k];
  U[d + 1] = p / (g - 1.0) + 0.5 * rho * v2;
}
// directional physical flux f(U, n) = sum_m n_m f_m(U)
void euler_flux(int d, double g, const double* U, const double* nv, double* F) {
  Prim s = prim(d, g, U);
  double vn = 0.0;
  for (int k = 0; k < d; ++k) vn += s.v[k] * nv[k];
  F[0] = s.rho * vn;
  for (int k = 0; k < d; ++k) F[1 + k] = s.rho * s.v[k] * vn + s.p * nv[k];
  F[d + 1] = vn * (U[d + 1] + s.p);
}

// logarithmic mean and its reciprocal, Taylor branch per R5.
thread_local int64_t tl_series = 0, tl_log = 0;
double ln_mean(double x, double y) {
  double f2 = (x * (x - 2.0 * y) + y * y) / (x * (x + 2.0 * y) + y * y);
  if (f2 < 1e-4) {
    ++tl_series;
    return (x + y) / (2.0 + f2 * (2.0 / 3.0 + f2 * (2.0 / 5.0 + f2 * (2.0 / 7.0))));
  }
  ++tl_log;
  return (y - x) / std::log(y / x);
}
double inv_ln_mean(double x, double y) {
  double f2 = (x * (x - 2.0 * y) + y * y) / (x * (x + 2.0 * y) + y * y);
  if (f2 < 1e-4) {
    ++tl_series;
    return (2.0 + f2 * (2.0 / 3.0 + f2 * (2.0 / 5.0 + f2 * (2.0 / 7.0)))) / (x + y);
  }
  ++tl_log;
  return std::log(y / x) / (y - x);
}

// Ranocha's entropy-conservative flux (P:834 [eq:ranocha_flux], energy component per R3) in
// directional form f#(a, b, n) = sum_m n_m f#_m(a, b).
void ec_flux(int d, double g, const double* Ua, const double* Ub, const double* nv, double* F) {
  Prim a = prim(d, g, Ua), b = prim(d, g, Ub);
  double rho_ln = ln_mean(a.rho, b.rho);
  double inv_beta_ln = inv_ln_mean(a.rho / a.p, b.rho / b.p);  // 1/<rho/p>_ln
  double vavg[3], vn = 0.0, vavg_n = 0.0, vavb_n = 0.0, vdot = 0.0;
  for (int k = 0; k < d; ++k) {
    vavg[k] = 0.5 * (a.v[k] + b.v[k]);
    vn += vavg[k] * nv[k];
    vavg_n += a.v[k] * nv[k];
    vavb_n += b.v[k] * nv[k];
    vdot += a.v[k] * b.v[k];
  }
  double pavg = 0.5 * (a.p + b.p);
  double fr = rho_ln * vn;
  F[0] = fr;
  for (int k = 0; k < d; ++k) F[1 + k] = fr * vavg[k] + pavg * nv[k];
  F[d + 1] = fr * (0.5 * vdot + inv_beta_ln / (g - 1.0)) + 0.5 * (a.p * vavb_n + b.p * vavg_n);
}
// Davis wave speed (P:839 [eq:wave_speed]) with a unit normal
double wave_speed(int d, double g, const double* Ua, const double* Ub, const double* nu) {
  Prim a = prim(d, g, Ua), b = prim(d, g, Ub);
  double va = 0.0, vb = 0.0;
  for (int k = 0; k < d; ++k) {
    va += a.v[k] * nu[k];
    vb += b.v[k] * nu[k];
  }
  return std::max(std::fabs(va), std::fabs(vb)) +
         std::max(std::sqrt(g * a.p / a.rho), std::sqrt(g * b.p / b.rho));
}
// entropy-stable interface flux (P:491 [eq:num_flux]) with a unit normal
void es_flux(int d, double g, const double* Ua, const double* Ub, const double* nu, double* F) {
  ec_flux(d, g, Ua, Ub, nu, F);
  double lam = wave_speed(d, g, Ua, Ub, nu);
  for (int e = 0; e < d + 2; ++e) F[e] -= 0.5 * lam * (Ub[e] - Ua[e]);
}

// du/dw at the state U: the inverse of the Hessian of S = -rho s/(g-1), symmetric positive
// definite for rho, p > 0 (Harten / Barth form; reading R27):
//   [ rho      rho v^T                E            ]
//   [ rho v    rho v v^T + p I        rho h v      ]     h = (E + p)/rho, a^2 = g p / rho
//   [ E        rho h v^T              rho h^2 - a^2 p/(g-1) ]
void dudw(int d, double g, const double* U, double* A /*[(d+2)^2] row-major*/) {
  Prim s = prim(d, g, U);
  int n = d + 2;
  double E = U[d + 1], h = (E + s.p) / s.rho, a2 = g * s.p / s.rho;
  A[0] = s.rho;
  for (int k = 0; k < d; ++k) A[1 + k] = A[(1 + k) * n] = s.rho * s.v[k];
  A[d + 1] = A[(d + 1) * n] = E;
  for (int k = 0; k < d; ++k) {
    for (int l = 0; l < d; ++l) A[(1 + k) * n + 1 + l] = s.rho * s.v[k] * s.v[l] + (k == l ? s.p : 0.0);
    A[(1 + k) * n + d + 1] = A[(d + 1) * n + 1 + k] = s.rho * h * s.v[k];
  }
  A[(d + 1) * n + d + 1] = s.rho * h * h - a2 * s.p / (g - 1.0);
}
// entropy-stable interface flux with scalar dissipation on the jump of the entropy variables
// (the alternative named at P:497, after Chandrashekar; reading R27):
//   f* = f#(Ua, Ub, n) - lambda/2 (du/dw)(U(wbar)) (w(Ub) - w(Ua)),  wbar = (w(Ua) + w(Ub))/2,
// lambda = Davis's wave speed.  du/dw is symmetric positive definite, so the dissipation
// removes entropy: [w]^T (f* - f#) = -lambda/2 [w]^T (du/dw) [w] <= 0.
void ej_flux(int d, double g, const double* Ua, const double* Ub, const double* nu, double* F) {
  ec_flux(d, g, Ua, Ub, nu, F);
  double lam = wave_speed(d, g, Ua, Ub, nu);
  int n = d + 2;
  double wa[5], wb[5], wm[5], Um[5], A[25];
  entropy_vars(d, g, Ua, wa);
  entropy_vars(d, g, Ub, wb);
  for (int e = 0; e < n; ++e) wm[e] = 0.5 * (wa[e] + wb[e]);
  cons_from_entropy(d, g, wm, Um);
  dudw(d, g, Um, A);
  for (int e = 0; e < n; ++e) {
    double t = 0.0;
    for (int k = 0; k < n; ++k) t += A[e * n + k] * (wb[k] - wa[k]);
    F[e] -= 0.5 * lam * t;
  }
}
// entropy-stable matrix dissipation (the alternative named at P:497, after Ismail-Roe / Winters et
// al.; reading R28): f* = f#(Ua, Ub, n) - 1/2 |A_n| (du/dw) [w], the normal flux Jacobian A_n and du/dw
// both at U(wbar).  With the eigenvectors of A_n scaled so that R T R^T = du/dw (Barth),
//   |A_n| du/dw = |v.n| du/dw + sum_{+,-} (|v.n +- a| - |v.n|) rho/(2g) r_+- r_+-^T,
//   r_+- = (1, v +- a n, h +- a v.n),  a^2 = g p / rho,  h = (E + p)/rho.
void md_flux(int d, double g, const double* Ua, const double* Ub, const double* nu, double* F) {
  ec_flux(d, g, Ua, Ub, nu, F);
  int n = d + 2;
  double wa[5], wb[5], wm[5], Um[5], A[25], dw[5];
  entropy_vars(d, g, Ua, wa);
  entropy_vars(d, g, Ub, wb);
  for (int e = 0; e < n; ++e) {
    wm[e] = 0.5 * (wa[e] + wb[e]);
    dw[e] = wb[e] - wa[e];
  }
  cons_from_entropy(d, g, wm, Um);
  dudw(d, g, Um, A);
  Prim s = prim(d, g, Um);
  double a = std::sqrt(g * s.p / s.rho), h = (Um[d + 1] + s.p) / s.rho, vn = 0.0;
  for (int k = 0; k < d; ++k) vn += s.v[k] * nu[k];
  double rm[5], rp[5];
  rm[0] = rp[0] = 1.0;
  for (int k = 0; k < d; ++k) {
    rm[1 + k] = s.v[k] - a * nu[k];
    rp[1 + k] = s.v[k] + a * nu[k];
  }
  rm[d + 1] = h - a * vn;
  rp[d + 1] = h + a * vn;
  double cm = (std::fabs(vn - a) - std::fabs(vn)) * s.rho / (2.0 * g);
  double cp = (std::fabs(vn + a) - std::fabs(vn)) * s.rho / (2.0 * g);
  double pm = 0.0, pp = 0.0;
  for (int e = 0; e < n; ++e) {
    pm += rm[e] * dw[e];
    pp += rp[e] * dw[e];
  }
  for (int e = 0; e < n; ++e) {
    double t = 0.0;
    for (int k = 0; k < n; ++k) t += A[e * n + k] * dw[k];
    F[e] -= 0.5 * (std::fabs(vn) * t + cm * pm * rm[e] + cp * pp * rp[e]);
  }
}
// interface flux by mode: 0 = entropy conservative, 1 = local Lax-Friedrichs,
// 2 = entropy-jump scalar dissipation (R27), 3 = matrix dissipation (R28)
void iface_flux(int mode, int d, double g, const double* Ua, const double* Ub, const double* nu, double* F) {
  if (mode == 1)
    es_flux(d, g, Ua, Ub, nu, F);
  else if (mode == 2)
    ej_flux(d, g, Ua, Ub, nu, F);
  else if (mode == 3)
    md_flux(d, g, Ua, Ub, nu, F);
  else
    ec_flux(d, g, Ua, Ub, nu, F);
}

// ------------------------------------------------------------------------------------------------
// small dense linear algebra: Gaussian elimination with partial pivoting, A X = B (in place)
// ------------------------------------------------------------------------------------------------
template <class T>
bool solve_dense(int N, vector<T> A, vector<T>& X, int nrhs) {
  for (int k = 0; k < N; ++k) {
    int piv = k;
    for (int i = k + 1; i < N; ++i)
      if (std::fabs(A[(size_t)i * N + k]) > std::fabs(A[(size_t)piv * N + k])) piv = i;
    if (A[(size_t)piv * N + k] == 0.0) return false;
    if (piv != k) {
      for (int j = 0; j < N; ++j) std::swap(A[(size_t)k * N + j], A[(size_t)piv * N + j]);
      for (int j = 0; j < nrhs; ++j) std::swap(X[(size_t)k * nrhs + j], X[(size_t)piv * nrhs + j]);
    }
    for (int i = k + 1; i < N; ++i) {
      T f = A[(size_t)i * N + k] / A[(size_t)k * N + k];
      if (f == 0.0) continue;
      for (int j = k; j < N; ++j) A[(size_t)i * N + j] -= f * A[(size_t)k * N + j];
      for (int j = 0; j < nrhs; ++j) X[(size_t)i * nrhs + j] -= f * X[(size_t)k * nrhs + j];
    }
  }
  for (int k = N - 1; k >= 0; --k) {
    for (int j = 0; j < nrhs; ++j) {
      T s = X[(size_t)k * nrhs + j];
      for (int i = k + 1; i < N; ++i) s -= A[(size_t)k * N + i] * X[(size_t)i * nrhs + j];
      X[(size_t)k * nrhs + j] = s / A[(size_t)k * N + k];
    }
  }
  return true;
}

// equispaced barycentric lattice of degree N on the reference simplex (R10)
// returns reference coordinates [M][d] and barycentric coordinates [M][d+1]
void lattice(int d, int N, vector<double>& xi, vector<double>& lam) {
  xi.clear();
  lam.clear();
  if (d == 2) {
    for (int j = 0; j <= N; ++j)
      for (int i = 0; i <= N - j; ++i) {
        double l2 = (double)i / N, l3 = (double)j / N;
        xi.push_back(-1.0 + 2.0 * l2);
        xi.push_back(-1.0 + 2.0 * l3);
        lam.push_back(1.0 - l2 - l3);
        lam.push_back(l2);
        lam.push_back(l3);
      }
  } else {
    for (int k = 0; k <= N; ++k)
      for (int j = 0; j <= N - k; ++j)
        for (int i = 0; i <= N - j - k; ++i) {
          double l2 = (double)i / N, l3 = (double)j / N, l4 = (double)k / N;
          xi.push_back(-1.0 + 2.0 * l2);
          xi.push_back(-1.0 + 2.0 * l3);
          xi.push_back(-1.0 + 2.0 * l4);
          lam.push_back(1.0 - l2 - l3 - l4);
          lam.push_back(l2);
          lam.push_back(l3);
          lam.push_back(l4);
        }
  }
}

// Geometry is evaluated in extended precision (long double, 64-bit significand): the equispaced
// lattice interpolation and differentiation of degree q+1 amplify rounding by ~1e3 (reading R25),
// so the oracle's metric terms are computed well below double-precision rounding and then rounded.
typedef long double LD;

// ---- warp & blend node family (P:845 names the interpolatory warp & blend of Chan & Warburton;
// reading R32: Warburton's warp & blend with the blending parameter alpha = 0) ----
// Gauss-Lobatto-Legendre points of degree N on [-1, 1], ascending: -1, the N - 1 roots of P_N', +1.
// Newton on P_N' from the Chebyshev-Gauss-Lobatto points, with P_N' and P_N'' from the Legendre
// recurrence and Legendre's equation (1 - x^2) P'' = 2 x P' - N (N + 1) P.
vector<LD> gll_points(int N) {
  vector<LD> x(N + 1);
  x[0] = -1.0L;
  x[N] = 1.0L;
  for (int i = 1; i < N; ++i) {
    LD t = -std::cos((LD)PI * (LD)i / (LD)N);
    for (int it = 0; it < 100; ++it) {
      LD p0 = 1.0L, p1 = t;  // P_0, P_1
      for (int k = 2; k <= N; ++k) {
        LD p2 = ((LD)(2 * k - 1) * t * p1 - (LD)(k - 1) * p0) / (LD)k;
        p0 = p1;
        p1 = p2;
      }
      // p1 = P_N, p0 = P_{N-1}
      LD dp = (LD)N * (t * p1 - p0) / (t * t - 1.0L);
      LD d2 = (2.0L * t * dp - (LD)N * (LD)(N + 1) * p1) / (1.0L - t * t);
      LD dt = dp / d2;
      t -= dt;
      if (std::fabs(dt) < 1e-19L) break;
    }
    x[i] = t;
  }
  return x;
}
// 1D warp factor (Warburton 2006): w(r) = sum_i (r_i^GLL - r_i^eq) l_i^eq(r), the degree-N interpolant on
// the equispaced points r_i^eq = -1 + 2i/N of the displacement to the GLL points, divided by 1 - r^2
// (w vanishes at +-1); 0 at |r| = 1 where the blend vanishes
LD warp_factor(int N, const vector<LD>& gll, LD r) {
  if (std::fabs(r) > 1.0L - 1e-12L) return 0.0L;
  LD w = 0.0L;
  for (int i = 0; i <= N; ++i) {
    LD ri = -1.0L + 2.0L * (LD)i / (LD)N, l = 1.0L;
    for (int j = 0; j <= N; ++j)
      if (j != i) {
        LD rj = -1.0L + 2.0L * (LD)j / (LD)N;
        l *= (r - rj) / (ri - rj);
      }
    w += (gll[i] - ri) * l;
  }
  return w / (1.0L - r * r);
}
// node family of degree N on the reference simplex: family 0 = the equispaced barycentric lattice
// (R10), family 1 = warp & blend (R32).  lam [M][d+1] barycentric coordinates (lam_1 = 1 - sum, vertex
// k+1 at xi_k = 1), xi [M][d] = -1 + 2 lam_{k+1}; same order as lattice().
//   2D: lam += sum over the edges (i, j) of 2 lam_i lam_j wf(lam_j - lam_i) (e_j - e_i) -- the edge
//       displacement w(r) along the edge, blended by 4 lam_i lam_j (= 1 - r^2 on the edge);
//   3D: per face F (the vertex a opposite), the face's 2D warp W_F in the raw barycentrics of its
//       vertices b, c, d, blended by lam_b lam_c lam_d / ((lam_b + lam_a/2)(lam_c + lam_a/2)(lam_d + lam_a/2));
//       nodes on an edge take W_F itself (the two faces through the edge agree there).
void node_set(int d, int N, int family, vector<LD>& xi, vector<LD>& lam) {
  vector<double> xid, lamd;
  lattice(d, N, xid, lamd);
  const int nb = d + 1, M = (int)lamd.size() / nb;
  lam.assign(lamd.size(), 0.0L);
  for (int i = 0; i < M; ++i) {  // exact lattice barycentrics k / N
    LD s = 0.0L;
    for (int k = 1; k < nb; ++k) {
      lam[(size_t)i * nb + k] = std::nearbyint(lamd[(size_t)i * nb + k] * N) / (LD)N;
      s += lam[(size_t)i * nb + k];
    }
    lam[(size_t)i * nb] = 1.0L - s;
  }
  if (family == 1 && N >= 3) {  // N <= 2: the GLL points are equispaced, no warp
    vector<LD> gll = gll_points(N);
    const LD tol = 1e-10L;
    for (int i = 0; i < M; ++i) {
      LD* L = &lam[(size_t)i * nb];
      LD shift[4] = {0, 0, 0, 0};
      auto face_warp = [&](const int* vs, int nvs, LD* W) {  // 2D warp of the vertices vs
        for (int k = 0; k < nb; ++k) W[k] = 0.0L;
        for (int x = 0; x < nvs; ++x)
          for (int y = x + 1; y < nvs; ++y) {
            int a = vs[x], b = vs[y];
            LD c = 2.0L * L[a] * L[b] * warp_factor(N, gll, L[b] - L[a]);
            W[b] += c;
            W[a] -= c;
          }
      };
      if (d == 2) {
        int vs[3] = {0, 1, 2};
        face_warp(vs, 3, shift);
      } else {
        for (int a = 0; a < 4; ++a) {
          int vs[3], q = 0;
          for (int k = 0; k < 4; ++k)
            if (k != a) vs[q++] = k;
          LD W[4];
          face_warp(vs, 3, W);
          LD lb = L[vs[0]], lc = L[vs[1]], ld = L[vs[2]], la = L[a];
          LD blend = lb * lc * ld, den = (lb + 0.5L * la) * (lc + 0.5L * la) * (ld + 0.5L * la);
          if (den > tol) blend /= den;
          for (int k = 0; k < 4; ++k) shift[k] += blend * W[k];
          int npos = (lb > tol) + (lc > tol) + (ld > tol);
          if (la < tol && npos < 3)
            for (int k = 0; k < 4; ++k) shift[k] = W[k];
        }
      }
      for (int k = 0; k < nb; ++k) L[k] += shift[k];
    }
  }
  xi.assign((size_t)M * d, 0.0L);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < d; ++k) xi[(size_t)i * d + k] = -1.0L + 2.0L * lam[(size_t)i * nb + k + 1];
}

// polynomial interpolant on a lattice in the PKD basis: coefficients for nrhs fields
struct Interp {
  int d, N, M;
  vector<int> al;
  vector<LD> xi;  // lattice points
  vector<LD> Vl;  // [M][M]
};
Interp make_interp(int d, int N, int family = 0) {
  Interp I;
  I.d = d;
  I.N = N;
  vector<LD> lamq;
  // interpolation points: the exact lattice coordinates -1 + 2 i/N in long double (family 0), or the
  // warp & blend points (family 1, R32)
  node_set(d, N, family, I.xi, lamq);
  I.al = multi_indices(d, N);
  I.M = (int)I.al.size() / d;
  I.Vl.assign((size_t)I.M * I.M, 0.0L);
  LD g[3];
  for (int i = 0; i < I.M; ++i)
    for (int k = 0; k < I.M; ++k) pkd_cart<LD>(d, &I.al[k * d], &I.xi[i * d], I.Vl[(size_t)i * I.M + k], g);
  return I;
}
// evaluate sum_k c[k][j] phi_k(x) and its gradient; c [M][nrhs]
void interp_eval(const Interp& I, const vector<LD>& c, int nrhs, const LD* x, LD* val, LD* grad /*[nrhs][d]*/) {
  int d = I.d;
  for (int j = 0; j < nrhs; ++j) {
    val[j] = 0.0;
    for (int k = 0; k < d; ++k) grad[j * d + k] = 0.0;
  }
  LD v, g[3];
  for (int k = 0; k < I.M; ++k) {
    pkd_cart<LD>(d, &I.al[k * d], x, v, g);
    for (int j = 0; j < nrhs; ++j) {
      LD ck = c[(size_t)k * nrhs + j];
      val[j] += ck * v;
      for (int l = 0; l < d; ++l) grad[j * d + l] += ck * g[l];
    }
  }
}

LD det_d(int d, const LD* A) {
  if (d == 2) return A[0] * A[3] - A[1] * A[2];
  return A[0] * (A[4] * A[8] - A[5] * A[7]) - A[1] * (A[3] * A[8] - A[5] * A[6]) +
         A[2] * (A[3] * A[7] - A[4] * A[6]);
}

}  // namespace

// ------------------------------------------------------------------------------------------------
// mesh + geometry
// ------------------------------------------------------------------------------------------------
struct ora_mesh {
  int d, p, Nc;
  double gamma;
  int64_t ne;
  Ref ref;
  vector<int64_t> ev;     // [ne][d+1]
  vector<double> evx;     // [ne][d+1][d]
  vector<double> period;  // [d]
  vector<char> has_geom;  // [ne]
  // per element geometry (empty for inactive elements)
  vector<vector<double>> G, Gf, Jt, Jn, xq;
  vector<int64_t> nbr;
  vector<int> nbr_face, reflect;
};

namespace {

// local vertices of facet z in (start, end, collapse) order (R11, derived from P:208-212)
void facet_verts(int d, int z, int* vs) {
  if (d == 2) {
    static const int t[3][2] = {{0, 1}, {1, 2}, {0, 2}};
    vs[0] = t[z][0];
    vs[1] = t[z][1];
  } else {
    static const int t[4][3] = {{0, 1, 3}, {1, 2, 3}, {0, 2, 3}, {0, 1, 2}};
    vs[0] = t[z][0];
    vs[1] = t[z][1];
    vs[2] = t[z][2];
  }
}

// geometry of one element (P:322-364 metric terms, P:448-452 Jacobian interpolant), evaluated in
// long double and rounded to double at the end (R25)
bool element_geometry(ora_mesh& m, int64_t el, const double* xmap /*[Npg][d]*/, const Interp& Ipg,
                      const Interp* Icurl) {
  const Ref& r = m.ref;
  int d = m.d, Nq = r.Nq, Nf = r.Nf, Nqf = r.Nqf;
  // interpolation coefficients of the mapping (P:327-331 [eq:poly_mapping])
  vector<LD> cx(xmap, xmap + (size_t)Ipg.M * d);
  if (!solve_dense<LD>(Ipg.M, Ipg.Vl, cx, d)) return false;
  vector<double> G((size_t)Nq * d * d), Gf((size_t)Nf * Nqf * d * d), Jt(Nq), Jn((size_t)Nf * Nqf * d),
      xq((size_t)Nq * d);
  LD val[3], A[9];
  auto gradx = [&](const LD* x, LD* vals, LD* Aout) {
    // Aout[mm*d + l] = d x_mm / d xi_l
    LD grad[9];
    interp_eval(Ipg, cx, d, x, vals, grad);
    for (int i = 0; i < d * d; ++i) Aout[i] = grad[i];
  };
  auto metric_at = [&](const LD* x, LD* Gout) {
    // exact metric terms = adjugate of the Jacobian, SURVEY App. B
    gradx(x, val, A);
    Gout[0] = A[3];   // G_11 = dx2/dxi2
    Gout[1] = -A[1];  // G_12 = -dx1/dxi2
    Gout[2] = -A[2];  // G_21 = -dx2/dxi1
    Gout[3] = A[0];   // G_22 = dx1/dxi1
  };
  // conservative curl metrics in 3D (P:349-356 [eq:metric_interpolants, eq:conservative_curl]),
  // column reading R4: G_{:,1} = -curl r1, G_{:,2} = curl r2, G_{:,3} = curl r3.
  vector<LD> cr;  // [Mcurl][9] coefficients of r1, r2, r3 (each 3 components)
  if (d == 3) {
    int Mc = Icurl->M;
    cr.assign((size_t)Mc * 9, 0.0L);
    for (int i = 0; i < Mc; ++i) {
      gradx(&Icurl->xi[i * 3], val, A);
      // r1 = x3 grad x2, r2 = x3 grad x1, r3 = x1 grad x2
      for (int l = 0; l < 3; ++l) {
        cr[(size_t)i * 9 + 0 + l] = val[2] * A[1 * 3 + l];
        cr[(size_t)i * 9 + 3 + l] = val[2] * A[0 * 3 + l];
        cr[(size_t)i * 9 + 6 + l] = val[0] * A[1 * 3 + l];
      }
    }
    if (!solve_dense<LD>(Mc, Icurl->Vl, cr, 9)) return false;
  }
  auto curl_metric_at = [&](const LD* x, LD* Gout) {
    LD v9[9], g27[27];
    interp_eval(*Icurl, cr, 9, x, v9, g27);
    // g27[(field)*3 + l] = d field / d xi_l, field = 3*rk + comp
    auto dr = [&](int rk, int comp, int l) { return g27[(3 * rk + comp) * 3 + l]; };
    for (int rk = 0; rk < 3; ++rk) {
      LD c0 = dr(rk, 2, 1) - dr(rk, 1, 2);
      LD c1 = dr(rk, 0, 2) - dr(rk, 2, 0);
      LD c2 = dr(rk, 1, 0) - dr(rk, 0, 1);
      LD s = (rk == 0) ? -1.0L : 1.0L;
      Gout[0 * 3 + rk] = s * c0;
      Gout[1 * 3 + rk] = s * c1;
      Gout[2 * 3 + rk] = s * c2;
    }
  };
  auto to_ld = [&](const double* x, LD* y) {
    for (int k = 0; k < d; ++k) y[k] = x[k];
  };
  for (int i = 0; i < Nq; ++i) {
    LD x[3], Gl[9], xv[3], gr[9];
    to_ld(&r.xi[i * d], x);
    if (d == 2)
      metric_at(x, Gl);
    else
      curl_metric_at(x, Gl);
    for (int k = 0; k < d * d; ++k) G[(size_t)i * d * d + k] = (double)Gl[k];
    interp_eval(Ipg, cx, d, x, xv, gr);
    for (int k = 0; k < d; ++k) xq[(size_t)i * d + k] = (double)xv[k];
  }
  for (int z = 0; z < Nf; ++z)
    for (int f = 0; f < Nqf; ++f) {
      LD x[3], Gl[9];
      to_ld(&r.xif[((size_t)z * Nqf + f) * d], x);
      if (d == 2)
        metric_at(x, Gl);
      else
        curl_metric_at(x, Gl);
      double* Go = &Gf[((size_t)z * Nqf + f) * d * d];
      for (int k = 0; k < d * d; ++k) Go[k] = (double)Gl[k];
      // J n = G^T nhat (P:361 [eq:nanson]); facet metric evaluated at the facet node (R8)
      for (int mm = 0; mm < d; ++mm) {
        LD s = 0.0;
        for (int l = 0; l < d; ++l) s += Gl[l * d + mm] * (LD)r.nhat[z * d + l];
        Jn[((size_t)z * Nqf + f) * d + mm] = (double)s;
      }
    }
  // Jacobian interpolant of degree p_g (P:448-452 [eq:jacobian_approx])
  vector<LD> cj(Ipg.M);
  for (int i = 0; i < Ipg.M; ++i) {
    gradx(&Ipg.xi[i * d], val, A);
    cj[i] = det_d(d, A);
    if (!(cj[i] > 0.0L)) {
      fprintf(stderr, "oracle: J <= 0 at mapping node %d of element %lld\n", i, (long long)el);
      return false;
    }
  }
  if (!solve_dense<LD>(Ipg.M, Ipg.Vl, cj, 1)) return false;
  for (int i = 0; i < Nq; ++i) {
    LD x[3], v1, g1[3];
    to_ld(&r.xi[i * d], x);
    interp_eval(Ipg, cj, 1, x, &v1, g1);
    Jt[i] = (double)v1;
    if (!(v1 > 0.0L)) {
      fprintf(stderr, "oracle: J~ <= 0 at volume node %d of element %lld\n", i, (long long)el);
      return false;
    }
  }
  for (int i = 0; i < Nq; ++i)  // back to global coordinates (R25)
    for (int k = 0; k < d; ++k) xq[(size_t)i * d + k] += m.evx[((size_t)el * (d + 1) + 0) * d + k];
  m.G[el] = G;
  m.Gf[el] = Gf;
  m.Jt[el] = Jt;
  m.Jn[el] = Jn;
  m.xq[el] = xq;
  m.has_geom[el] = 1;
  return true;
}

}  // namespace

extern "C" {

double ora_jacobi(int n, double a, double b, double x) { return jacobi(n, a, b, x); }
double ora_jacobi_deriv(int n, double a, double b, double x) { return jacobi_deriv(n, a, b, x); }
int ora_gauss_jacobi(int q, double a, double b, double* x, double* w) {
  vector<double> xs, ws;
  gauss_jacobi(q, a, b, xs, ws);
  for (int i = 0; i <= q; ++i) {
    x[i] = xs[i];
    w[i] = ws[i];
  }
  return 0;
}
void ora_lagrange_diff(int n, const double* nodes, double* D) {
  vector<double> nd(nodes, nodes + n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) D[i * n + j] = lagrange_deriv(nd, j, nd[i]);
}

void ora_ref_sizes(int d, int q, int p, int* out) {
  int n = q + 1;
  out[0] = n;
  out[1] = (d == 2) ? n * n : n * n * n;
  out[2] = d + 1;
  out[3] = (d == 2) ? n : n * n;
  out[4] = (int)multi_indices(d, p).size() / d;
}

int ora_ref_get(int d, int q, int p, const char* name, double* out) {
  Ref r = build_ref(d, q, p);
  std::string s(name);
  const vector<double>* src = nullptr;
  if (s == "eta1") src = &r.eta1;
  else if (s == "w1") src = &r.w1;
  else if (s == "eta3") src = &r.eta3;
  else if (s == "w3") src = &r.w3;
  else if (s == "xi") src = &r.xi;
  else if (s == "eta") src = &r.eta;
  else if (s == "W") src = &r.W;
  else if (s == "xif") src = &r.xif;
  else if (s == "B") src = &r.B;
  else if (s == "nhat") src = &r.nhat;
  else if (s == "D") src = &r.D;
  else if (s == "Q") src = &r.Q;
  else if (s == "E") src = &r.E;
  else if (s == "S") src = &r.S;
  else if (s == "R") src = &r.R;
  else if (s == "V") src = &r.V;
  else if (s == "alpha") {
    for (size_t k = 0; k < r.alpha.size(); ++k) out[k] = r.alpha[k];
    return 0;
  }
  if (!src) return -1;
  std::memcpy(out, src->data(), src->size() * sizeof(double));
  return 0;
}

void ora_pkd_eval(int d, int p, int npts, const double* xi, double* vals, double* grads) {
  vector<int> al = multi_indices(d, p);
  int Np = (int)al.size() / d;
  for (int i = 0; i < npts; ++i)
    for (int k = 0; k < Np; ++k) {
      double v, g[3];
      pkd_cart(d, &al[k * d], &xi[i * d], v, g);
      vals[(size_t)i * Np + k] = v;
      if (grads)
        for (int l = 0; l < d; ++l) grads[((size_t)i * Np + k) * d + l] = g[l];
    }
}

void ora_entropy_vars(int d, double g, int n, const double* U, double* W) {
  for (int i = 0; i < n; ++i) entropy_vars(d, g, U + (size_t)i * (d + 2), W + (size_t)i * (d + 2));
}
void ora_cons_from_entropy(int d, double g, int n, const double* W, double* U) {
  for (int i = 0; i < n; ++i) cons_from_entropy(d, g, W + (size_t)i * (d + 2), U + (size_t)i * (d + 2));
}
void ora_euler_flux(int d, double g, int n, const double* U, const double* nv, double* F) {
  for (int i = 0; i < n; ++i) euler_flux(d, g, U + (size_t)i * (d + 2), nv + (size_t)i * d, F + (size_t)i * (d + 2));
}
void ora_ec_flux(int d, double g, int n, const double* Ua, const double* Ub, const double* nv, double* F) {
  for (int i = 0; i < n; ++i)
    ec_flux(d, g, Ua + (size_t)i * (d + 2), Ub + (size_t)i * (d + 2), nv + (size_t)i * d, F + (size_t)i * (d + 2));
}
void ora_es_flux(int d, double g, int n, const double* Ua, const double* Ub, const double* nu, double* F) {
  for (int i = 0; i < n; ++i)
    es_flux(d, g, Ua + (size_t)i * (d + 2), Ub + (size_t)i * (d + 2), nu + (size_t)i * d, F + (size_t)i * (d + 2));
}
void ora_dudw(int d, double g, int n, const double* U, double* A) {
  for (int i = 0; i < n; ++i) dudw(d, g, U + (size_t)i * (d + 2), A + (size_t)i * (d + 2) * (d + 2));
}
void ora_ej_flux(int d, double g, int n, const double* Ua, const double* Ub, const double* nu, double* F) {
  for (int i = 0; i < n; ++i)
    ej_flux(d, g, Ua + (size_t)i * (d + 2), Ub + (size_t)i * (d + 2), nu + (size_t)i * d, F + (size_t)i * (d + 2));
}
void ora_md_flux(int d, double g, int n, const double* Ua, const double* Ub, const double* nu, double* F) {
  for (int i = 0; i < n; ++i)
    md_flux(d, g, Ua + (size_t)i * (d + 2), Ub + (size_t)i * (d + 2), nu + (size_t)i * d, F + (size_t)i * (d + 2));
}
double ora_wave_speed(int d, double g, const double* Ua, const double* Ub, const double* nu) {
  return wave_speed(d, g, Ua, Ub, nu);
}
double ora_ln_mean(double x, double y) { return ln_mean(x, y); }
double ora_inv_ln_mean(double x, double y) { return inv_ln_mean(x, y); }
void ora_entropy(int d, double g, int n, const double* U, double* S, double* Fent) {
  // S = -rho ln(p/rho^g)/(g-1), F = v S
  for (int i = 0; i < n; ++i) {
    Prim s = prim(d, g, U + (size_t)i * (d + 2));
    double Si = -s.rho * std::log(s.p / std::pow(s.rho, g)) / (g - 1.0);
    S[i] = Si;
    if (Fent)
      for (int k = 0; k < d; ++k) Fent[(size_t)i * d + k] = s.v[k] * Si;
  }
}

ora_mesh* ora_mesh_create(int d, int p, int64_t ne, const int64_t* elem_vertices,
                          const double* elem_vertex_coords, const double* period, ora_map_fn map,
                          void* user, double gamma, int64_t n_active, const int64_t* active) {
  return ora_mesh_create2(d, p, ne, elem_vertices, elem_vertex_coords, period, map, user, gamma, n_active, active, 0);
}

int ora_nodes(int d, int N, int family, double* xi, double* lam) {
  vector<LD> x, l;
  node_set(d, N, family, x, l);
  if (xi)
    for (size_t k = 0; k < x.size(); ++k) xi[k] = (double)x[k];
  if (lam)
    for (size_t k = 0; k < l.size(); ++k) lam[k] = (double)l[k];
  return (int)(l.size() / (d + 1));
}

ora_mesh* ora_mesh_create2(int d, int p, int64_t ne, const int64_t* elem_vertices,
                           const double* elem_vertex_coords, const double* period, ora_map_fn map,
                           void* user, double gamma, int64_t n_active, const int64_t* active, int node_family) {
  if (node_family < 0 || node_family > 1) return nullptr;
  ora_mesh* m = new ora_mesh();
  m->d = d;
  m->p = p;
  m->Nc = d + 2;
  m->gamma = gamma;
  m->ne = ne;
  m->ref = build_ref(d, p, p);  // q = p
  int nv = d + 1;
  m->ev.assign(elem_vertices, elem_vertices + ne * nv);
  m->evx.assign(elem_vertex_coords, elem_vertex_coords + ne * nv * d);
  m->period.assign(period, period + d);
  m->has_geom.assign(ne, 0);
  m->G.resize(ne);
  m->Gf.resize(ne);
  m->Jt.resize(ne);
  m->Jn.resize(ne);
  m->xq.resize(ne);
  const Ref& r = m->ref;
  int Nf = r.Nf;
  // ---- connectivity (Assumption P:736-741), orientation per R11 ----
  m->nbr.assign(ne * Nf, -1);
  m->nbr_face.assign(ne * Nf, -1);
  m->reflect.assign(ne * Nf, 0);
  std::map<vector<int64_t>, vector<std::pair<int64_t, int>>> faces;
  for (int64_t e = 0; e < ne; ++e)
    for (int z = 0; z < Nf; ++z) {
      int vs[3];
      facet_verts(d, z, vs);
      vector<int64_t> key;
      for (int k = 0; k < d; ++k) key.push_back(m->ev[e * nv + vs[k]]);
      std::sort(key.begin(), key.end());
      faces[key].push_back({e, z});
    }
  for (auto& kv : faces) {
    if (kv.second.size() != 2) {
      fprintf(stderr, "oracle: face shared by %zu elements (need a closed conforming mesh)\n",
              kv.second.size());
      delete m;
      return nullptr;
    }
    for (int s = 0; s < 2; ++s) {
      int64_t e = kv.second[s].first, o = kv.second[1 - s].first;
      int z = kv.second[s].second, zo = kv.second[1 - s].second;
      int va[3], vb[3];
      facet_verts(d, z, va);
      facet_verts(d, zo, vb);
      int64_t s0 = m->ev[e * nv + va[0]], s1 = m->ev[e * nv + va[1]];
      int64_t o0 = m->ev[o * nv + vb[0]], o1 = m->ev[o * nv + vb[1]];
      if (d == 3 && m->ev[e * nv + va[2]] != m->ev[o * nv + vb[2]]) {
        fprintf(stderr, "oracle: collapse vertices differ on a face of element %lld\n", (long long)e);
        delete m;
        return nullptr;
      }
      m->nbr[e * Nf + z] = o;
      m->nbr_face[e * Nf + z] = zo;
      if (s0 == o0 && s1 == o1)
        m->reflect[e * Nf + z] = 0;
      else if (s0 == o1 && s1 == o0)
        m->reflect[e * Nf + z] = 1;
      else {
        fprintf(stderr, "oracle: inconsistent face orientation\n");
        delete m;
        return nullptr;
      }
    }
  }
  // ---- active set: requested elements plus their face neighbours ----
  vector<char> act(ne, 0);
  if (!active) {
    std::fill(act.begin(), act.end(), 1);
  } else {
    for (int64_t i = 0; i < n_active; ++i) {
      int64_t e = active[i];
      act[e] = 1;
      for (int z = 0; z < Nf; ++z) act[m->nbr[e * Nf + z]] = 1;
    }
  }
  vector<int64_t> alist;
  for (int64_t e = 0; e < ne; ++e)
    if (act[e]) alist.push_back(e);
  // ---- mapping nodes: affine images of the degree-p_g lattice, then the user map ----
  Interp Ipg = make_interp(d, p, node_family);
  Interp Icurl;
  if (d == 3) Icurl = make_interp(d, p + 1, node_family);  // curl interpolation of degree q+1
  vector<LD> lxiq, llamq;
  node_set(d, p, node_family, lxiq, llamq);
  vector<double> llam(llamq.begin(), llamq.end());
  int Npg = Ipg.M;
  vector<double> xin((size_t)alist.size() * Npg * d), xout(xin.size());
  for (size_t a = 0; a < alist.size(); ++a) {
    int64_t e = alist[a];
    for (int i = 0; i < Npg; ++i)
      for (int k = 0; k < d; ++k) {
        double s = 0.0;
        for (int v = 0; v < nv; ++v) s += llam[(size_t)i * nv + v] * m->evx[(e * nv + v) * d + k];
        xin[((size_t)a * Npg + i) * d + k] = s;
      }
  }
  if (map)
    map(user, (int64_t)alist.size() * Npg, xin.data(), xout.data());
  else
    xout = xin;
  // geometry in element-local coordinates x - X_1 (reading R25: G, J and J~ are invariant under a
  // translation of the map -- for the curl form because curl I_{q+1}[c grad x_k] = c curl grad x_k
  // = 0 exactly, grad x_k being in P_{p-1} -- and local coordinates avoid cancellation of size L/h)
  for (size_t a = 0; a < alist.size(); ++a)
    for (int i = 0; i < Npg; ++i)
      for (int k = 0; k < d; ++k) xout[((size_t)a * Npg + i) * d + k] -= m->evx[(alist[a] * nv + 0) * d + k];
  bool ok = true;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t a = 0; a < (int64_t)alist.size(); ++a) {
    if (!element_geometry(*m, alist[a], &xout[(size_t)a * Npg * d], Ipg, d == 3 ? &Icurl : nullptr)) {
#pragma omp critical
      ok = false;
    }
  }
  if (!ok) {
    delete m;
    return nullptr;
  }
  // ---- geometric validation of the pairing (P:736-741 [eq:weights_match]) ----
  int Nqf = r.Nqf, n = r.n;
  for (int64_t e : alist)
    for (int z = 0; z < Nf; ++z) {
      int64_t o = m->nbr[e * Nf + z];
      if (!m->has_geom[o]) continue;
      int zo = m->nbr_face[e * Nf + z], rf = m->reflect[e * Nf + z];
      for (int f = 0; f < Nqf; ++f) {
        int i1 = f % n, i2 = f / n;
        int fo = (d == 2) ? (rf ? n - 1 - f : f) : ((rf ? n - 1 - i1 : i1) + n * i2);
        // normals equal and opposite, omega J_f equal
        double s2 = 0.0, na = 0.0;
        for (int k = 0; k < d; ++k) {
          double a = m->Jn[e][((size_t)z * Nqf + f) * d + k] * r.B[z * Nqf + f];
          double b = m->Jn[o][((size_t)zo * Nqf + fo) * d + k] * r.B[zo * Nqf + fo];
          s2 += (a + b) * (a + b);
          na += a * a;
        }
        if (std::sqrt(s2) > 1e-8 * std::sqrt(na)) {
          fprintf(stderr, "oracle: face normals of element %lld facet %d do not match (%g)\n",
                  (long long)e, z + 1, std::sqrt(s2 / na));
          ok = false;
        }
      }
    }
  if (!ok) {
    delete m;
    return nullptr;
  }
  return m;
}

void ora_mesh_destroy(ora_mesh* m) { delete m; }

int ora_mesh_geometry(const ora_mesh* m, int64_t el, double* G, double* Gf, double* Jt, double* Jn,
                      double* xq) {
  if (el < 0 || el >= m->ne || !m->has_geom[el]) return -1;
  if (G) std::memcpy(G, m->G[el].data(), m->G[el].size() * 8);
  if (Gf) std::memcpy(Gf, m->Gf[el].data(), m->Gf[el].size() * 8);
  if (Jt) std::memcpy(Jt, m->Jt[el].data(), m->Jt[el].size() * 8);
  if (Jn) std::memcpy(Jn, m->Jn[el].data(), m->Jn[el].size() * 8);
  if (xq) std::memcpy(xq, m->xq[el].data(), m->xq[el].size() * 8);
  return 0;
}

// Modal (compressed) metric storage ("the only necessary storage being
// geometric information", stored here as PKD coefficients instead of nodal values).  The metric
// terms are polynomials of degree <= p in the reference coordinates: in 2D the exact metrics of the
// degree-p_g = p map have degree p - 1, in 3D the conservative curl form differentiates
// the degree-(q+1) interpolant once (R4), degree q = p.  With M = V^T W V = I the
// L2 projection g~ = V^T W G is therefore exact and V g~ reproduces G at the volume nodes (up to
// rounding).  g~ [d*d][Np]: row l*d + m holds G_lm.
int ora_metric_modal(const ora_mesh* m, int64_t el, double* gm) {
  if (el < 0 || el >= m->ne || !m->has_geom[el]) return -1;
  const Ref& r = m->ref;
  const int d = m->d, Nq = r.Nq, Np = r.Np;
  const vector<double>& G = m->G[el];  // [Nq][d][d]
  for (int lm = 0; lm < d * d; ++lm)
    for (int k = 0; k < Np; ++k) {
      double s = 0.0;  // (V^T W G_lm)_k
      for (int i = 0; i < Nq; ++i) s += r.V[(size_t)i * Np + k] * r.W[i] * G[(size_t)i * d * d + lm];
      gm[(size_t)lm * Np + k] = s;
    }
  return 0;
}

int ora_mesh_use_modal_metrics(ora_mesh* m) {
  const Ref& r = m->ref;
  const int d = m->d, Nq = r.Nq, Np = r.Np;
  vector<double> gm((size_t)d * d * Np);
  for (int64_t el = 0; el < m->ne; ++el) {
    if (!m->has_geom[el]) continue;
    ora_metric_modal(m, el, gm.data());
    vector<double>& G = m->G[el];
    for (int i = 0; i < Nq; ++i)
      for (int lm = 0; lm < d * d; ++lm) {
        double s = 0.0;  // (V g~_lm)_i
        for (int k = 0; k < Np; ++k) s += r.V[(size_t)i * Np + k] * gm[(size_t)lm * Np + k];
        G[(size_t)i * d * d + lm] = s;
      }
  }
  return 0;
}

void ora_mesh_conn(const ora_mesh* m, int64_t* nbr, int* nbr_face, int* reflect) {
  size_t N = m->nbr.size();
  for (size_t i = 0; i < N; ++i) {
    nbr[i] = m->nbr[i];
    nbr_face[i] = m->nbr_face[i];
    reflect[i] = m->reflect[i];
  }
}

void ora_project(const ora_mesh* m, int64_t n_el, const int64_t* elems, const double* u_nodal,
                 double* u_modal) {
  const Ref& r = m->ref;
  int Nq = r.Nq, Np = r.Np, Nc = m->Nc;
  for (int64_t a = 0; a < n_el; ++a) {
    int64_t e = elems[a];
    for (int c = 0; c < Nc; ++c)
      for (int k = 0; k < Np; ++k) {
        double s = 0.0;  // (V^T W u)_k, reference L2 projection with M = I (R18)
        for (int i = 0; i < Nq; ++i)
          s += r.V[(size_t)i * Np + k] * r.W[i] * u_nodal[((size_t)e * Nq + i) * Nc + c];
        u_modal[((size_t)e * Nc + c) * Np + k] = s;
      }
  }
}

}  // extern "C"

// ------------------------------------------------------------------------------------------------
// the right-hand side
// ------------------------------------------------------------------------------------------------
namespace {

struct Proj {  // entropy-projected quantities of one element
  vector<double> w;    // [Nq][Nc] projected entropy variables at volume nodes
  vector<double> ub;   // [Nq][Nc] entropy-projected conservative variables U(w)
  vector<double> ubf;  // [Nf][Nqf][Nc] U(w_f) at facet nodes
  bool admissible;
};

// y = V x  (x [Np], y [Nq]) and y = V^T x, dense
void Vapply(const Ref& r, const double* x, double* y) {
  for (int i = 0; i < r.Nq; ++i) {
    double s = 0.0;
    for (int k = 0; k < r.Np; ++k) s += r.V[(size_t)i * r.Np + k] * x[k];
    y[i] = s;
  }
}
void VTapply(const Ref& r, const double* x, double* y) {
  for (int k = 0; k < r.Np; ++k) {
    double s = 0.0;
    for (int i = 0; i < r.Nq; ++i) s += r.V[(size_t)i * r.Np + k] * x[i];
    y[k] = s;
  }
}
// weight-adjusted inverse applied to V^T y: M~^{-1} V^T y = V^T W/J~ V (V^T y) with M = I
// (P:441-447 [eq:weight_adjusted_inverse], P:593 [eq:matvec_dudt])
void wadg(const ora_mesh& m, int64_t e, const double* ynodal, double* out) {
  const Ref& r = m.ref;
  vector<double> t1(r.Np), t2(r.Nq);
  VTapply(r, ynodal, t1.data());
  Vapply(r, t1.data(), t2.data());
  for (int i = 0; i < r.Nq; ++i) t2[i] *= r.W[i] / m.Jt[e][i];
  VTapply(r, t2.data(), out);
}

bool prim_ok(int d, double g, const double* U) {
  if (!(U[0] > 0.0)) return false;
  Prim s = prim(d, g, U);
  return s.p > 0.0;
}

Proj project(const ora_mesh& m, int64_t e, const double* ue /*[Nc][Np]*/) {
  const Ref& r = m.ref;
  int d = m.d, Nq = r.Nq, Np = r.Np, Nc = m.Nc, Nf = r.Nf, Nqf = r.Nqf;
  double g = m.gamma;
  Proj P;
  P.admissible = true;
  // u = V u~ (P:583 [eq:matvec_cons_vars])
  vector<double> u((size_t)Nq * Nc), tmp(Nq);
  for (int c = 0; c < Nc; ++c) {
    Vapply(r, ue + (size_t)c * Np, tmp.data());
    for (int i = 0; i < Nq; ++i) u[(size_t)i * Nc + c] = tmp[i];
  }
  // entropy variables at volume nodes, W(u_i)
  vector<double> Wn((size_t)Nq * Nc);
  for (int i = 0; i < Nq; ++i) {
    if (!prim_ok(d, g, &u[(size_t)i * Nc])) {
      P.admissible = false;
      return P;
    }
    entropy_vars(d, g, &u[(size_t)i * Nc], &Wn[(size_t)i * Nc]);
  }
  // w~ = M^{-1} V^T W J~^{-1} V M^{-1} V^T W J~ W(u)  (P:586 [eq:matvec_entropy_projection], R6)
  P.w.assign((size_t)Nq * Nc, 0.0);
  vector<double> y(Nq), wt(Np), wn(Nq);
  for (int c = 0; c < Nc; ++c) {
    for (int i = 0; i < Nq; ++i) y[i] = r.W[i] * m.Jt[e][i] * Wn[(size_t)i * Nc + c];
    wadg(m, e, y.data(), wt.data());
    Vapply(r, wt.data(), wn.data());  // w = V w~
    for (int i = 0; i < Nq; ++i) P.w[(size_t)i * Nc + c] = wn[i];
  }
  // facet values w_f = R^(z) w
  vector<double> wf((size_t)Nf * Nqf * Nc, 0.0);
  for (int z = 0; z < Nf; ++z)
    for (int f = 0; f < Nqf; ++f)
      for (int c = 0; c < Nc; ++c) {
        double s = 0.0;
        for (int i = 0; i < Nq; ++i) s += r.R[((size_t)z * Nqf + f) * Nq + i] * P.w[(size_t)i * Nc + c];
        wf[((size_t)z * Nqf + f) * Nc + c] = s;
      }
  // entropy-projected conservative variables
  P.ub.assign((size_t)Nq * Nc, 0.0);
  P.ubf.assign((size_t)Nf * Nqf * Nc, 0.0);
  for (int i = 0; i < Nq; ++i) {
    if (!(P.w[(size_t)i * Nc + d + 1] < 0.0)) P.admissible = false;
    cons_from_entropy(d, g, &P.w[(size_t)i * Nc], &P.ub[(size_t)i * Nc]);
    if (!prim_ok(d, g, &P.ub[(size_t)i * Nc])) P.admissible = false;
  }
  for (int k = 0; k < Nf * Nqf; ++k) {
    if (!(wf[(size_t)k * Nc + d + 1] < 0.0)) P.admissible = false;
    cons_from_entropy(d, g, &wf[(size_t)k * Nc], &P.ubf[(size_t)k * Nc]);
    if (!prim_ok(d, g, &P.ubf[(size_t)k * Nc])) P.admissible = false;
  }
  return P;
}

struct ElemOut {
  int64_t vp = 0, fp = 0, ie = 0, ser = 0, lg = 0;
  double erate = 0.0, eabs = 0.0, cons[5] = {0, 0, 0, 0, 0};
  bool admissible = true;
};

// nodal residual r of one element (P:520 [eq:entropy_stable], P:525 [eq:facet_correction]) and
// dudt = M~^{-1} V^T r (P:446 [eq:dudt_modal]).
void element_rhs(const ora_mesh& m, int64_t e, const vector<Proj>& PJ, const vector<int64_t>& slot,
                 int flux_mode, int variant, double* dudt, ElemOut& out) {
  const Ref& r = m.ref;
  int d = m.d, Nq = r.Nq, Nc = m.Nc, Nf = r.Nf, Nqf = r.Nqf, n = r.n;
  double g = m.gamma;
  const Proj& P = PJ[slot[e]];
  const vector<double>& G = m.G[e];
  int64_t s0 = tl_series, l0 = tl_log;
  vector<double> res((size_t)Nq * Nc, 0.0);  // r
  double F[5], nv[3];
  auto gvec = [&](int i, int l, double* gout) {  // g^(l) = row l of G at volume node i
    for (int mm = 0; mm < d; ++mm) gout[mm] = G[((size_t)i * d + l) * d + mm];
  };
  double gi[3], gj[3];
  if (variant == 3) {
    // ---- hybridised SBP formulation, Chan-Wilcox eq. (35) ----
    int Nb = Nq + Nf * Nqf;
    // hybridised reference operators Q-bar^(l) (P:648 [eq:q_hybridized])
    vector<double> Qb((size_t)d * Nb * Nb, 0.0);
    for (int l = 0; l < d; ++l) {
      double* Ql = &Qb[(size_t)l * Nb * Nb];
      for (int i = 0; i < Nq; ++i)
        for (int j = 0; j < Nq; ++j) Ql[(size_t)i * Nb + j] = r.S[((size_t)l * Nq + i) * Nq + j];
      for (int z = 0; z < Nf; ++z) {
        double nl = r.nhat[z * d + l];
        for (int f = 0; f < Nqf; ++f) {
          int jf = Nq + z * Nqf + f;
          double bf = r.B[z * Nqf + f];
          for (int i = 0; i < Nq; ++i) {
            double rb = r.R[((size_t)z * Nqf + f) * Nq + i] * bf;
            Ql[(size_t)i * Nb + jf] = 0.5 * nl * rb;
            Ql[(size_t)jf * Nb + i] = -0.5 * nl * rb;
          }
          Ql[(size_t)jf * Nb + jf] = 0.5 * nl * bf;
        }
      }
    }
    // hybridised states and metric terms (volume, then facets)
    vector<double> ubar((size_t)Nb * Nc), Gb((size_t)Nb * d * d);
    for (int i = 0; i < Nq; ++i) {
      for (int c = 0; c < Nc; ++c) ubar[(size_t)i * Nc + c] = P.ub[(size_t)i * Nc + c];
      for (int k = 0; k < d * d; ++k) Gb[(size_t)i * d * d + k] = G[(size_t)i * d * d + k];
    }
    for (int k = 0; k < Nf * Nqf; ++k) {
      for (int c = 0; c < Nc; ++c) ubar[(size_t)(Nq + k) * Nc + c] = P.ubf[(size_t)k * Nc + c];
      for (int kk = 0; kk < d * d; ++kk) Gb[(size_t)(Nq + k) * d * d + kk] = m.Gf[e][(size_t)k * d * d + kk];
    }
    // sum_m (2 Qbar^(k,m) o Fbar^(m)) 1, Qbar^(k,m) = sum_l Qbar^(l) o <Gbar_lm>
    vector<double> y((size_t)Nb * Nc, 0.0);
    for (int i = 0; i < Nb; ++i)
      for (int j = 0; j < Nb; ++j) {
        double qm[3] = {0, 0, 0};
        bool any = false;
        for (int mm = 0; mm < d; ++mm) {
          for (int l = 0; l < d; ++l) {
            double q = Qb[((size_t)l * Nb + i) * Nb + j];
            if (q == 0.0) continue;
            qm[mm] += q * 0.5 * (Gb[(size_t)i * d * d + l * d + mm] + Gb[(size_t)j * d * d + l * d + mm]);
          }
          if (qm[mm] != 0.0) any = true;
        }
        if (!any) continue;
        // sum_m 2 Qbar_ij^(m) f#_m(u_i, u_j) = f#(u_i, u_j, 2 qm) by linearity in n
        for (int mm = 0; mm < d; ++mm) nv[mm] = 2.0 * qm[mm];
        ec_flux(d, g, &ubar[(size_t)i * Nc], &ubar[(size_t)j * Nc], nv, F);
        out.vp++;
        for (int c = 0; c < Nc; ++c) y[(size_t)i * Nc + c] += F[c];
      }
    // z = -(y_vol + sum R^T y_f) - sum R^T B J_f (f* - sum_m N_m f_m(u_f))
    for (int i = 0; i < Nq; ++i)
      for (int c = 0; c < Nc; ++c) res[(size_t)i * Nc + c] = -y[(size_t)i * Nc + c];
    for (int z = 0; z < Nf; ++z) {
      int64_t o = m.nbr[e * Nf + z];
      int zo = m.nbr_face[e * Nf + z], rf = m.reflect[e * Nf + z];
      const Proj& PO = PJ[slot[o]];
      for (int f = 0; f < Nqf; ++f) {
        int i1 = f % n, i2 = f / n;
        int fo = (d == 2) ? (rf ? n - 1 - f : f) : ((rf ? n - 1 - i1 : i1) + n * i2);
        const double* um = &P.ubf[((size_t)z * Nqf + f) * Nc];
        const double* up = &PO.ubf[((size_t)zo * Nqf + fo) * Nc];
        const double* Jn = &m.Jn[e][((size_t)z * Nqf + f) * d];
        double Jf = 0.0;
        for (int k = 0; k < d; ++k) Jf += Jn[k] * Jn[k];
        Jf = std::sqrt(Jf);
        double nu[3];
        for (int k = 0; k < d; ++k) nu[k] = Jn[k] / Jf;
        double fs[5], fphys[5];
        iface_flux(flux_mode, d, g, um, up, nu, fs);
        out.ie++;
        euler_flux(d, g, um, nu, fphys);
        double bf = r.B[z * Nqf + f];
        for (int c = 0; c < Nc; ++c) {
          double sv = y[(size_t)(Nq + z * Nqf + f) * Nc + c] + bf * Jf * (fs[c] - fphys[c]);
          for (int i = 0; i < Nq; ++i) res[(size_t)i * Nc + c] -= r.R[((size_t)z * Nqf + f) * Nq + i] * sv;
        }
      }
    }
  } else {
    // ---- volume flux differencing (P:520 first line; P:541-547 [eq:flux_differencing]) ----
    if (variant == 0 || variant == 2) {
      for (int l = 0; l < d; ++l) {
        const double* Sl = &r.S[(size_t)l * Nq * Nq];
        double smax = 0.0;
        for (size_t k = 0; k < (size_t)Nq * Nq; ++k) smax = std::max(smax, std::fabs(Sl[k]));
        for (int i = 0; i < Nq; ++i) {
          int j0 = (variant == 0) ? i + 1 : 0;
          for (int j = j0; j < Nq; ++j) {
            double s = Sl[(size_t)i * Nq + j];
            if (variant == 0 && !(std::fabs(s) > 1e-12 * smax)) continue;  // structural nnz (R19)
            gvec(i, l, gi);
            gvec(j, l, gj);
            for (int mm = 0; mm < d; ++mm) nv[mm] = gi[mm] + gj[mm];  // <2 g^(l)>_ij
            ec_flux(d, g, &P.ub[(size_t)i * Nc], &P.ub[(size_t)j * Nc], nv, F);
            out.vp++;
            for (int c = 0; c < Nc; ++c) {
              res[(size_t)i * Nc + c] -= s * F[c];
              if (variant == 0) res[(size_t)j * Nc + c] += s * F[c];  // skew-symmetry of S
            }
          }
        }
      }
    } else {
      // line-wise pairing in collapsed coordinates: one flux per pair on each eta_k-line,
      // with n_ij = sum_l S^(l)_ij (g_i^(l) + g_j^(l)) (f# is linear in its direction argument)
      int nlines = (d == 2) ? n : n * n;
      for (int k = 0; k < d; ++k)
        for (int L = 0; L < nlines; ++L)
          for (int a = 0; a < n; ++a)
            for (int b = a + 1; b < n; ++b) {
              int idx[3], jdx[3];
              int o1 = L % n, o2 = L / n;
              // line along direction k with the other indices fixed
              int pos = 0;
              int other[2] = {o1, o2};
              for (int t = 0; t < d; ++t) {
                if (t == k) {
                  idx[t] = a;
                  jdx[t] = b;
                } else {
                  idx[t] = other[pos];
                  jdx[t] = other[pos];
                  ++pos;
                }
              }
              int i = idx[0] + n * idx[1] + (d == 3 ? n * n * idx[2] : 0);
              int j = jdx[0] + n * jdx[1] + (d == 3 ? n * n * jdx[2] : 0);
              for (int mm = 0; mm < d; ++mm) nv[mm] = 0.0;
              for (int l = 0; l < d; ++l) {
                double s = r.S[((size_t)l * Nq + i) * Nq + j];
                gvec(i, l, gi);
                gvec(j, l, gj);
                for (int mm = 0; mm < d; ++mm) nv[mm] += s * (gi[mm] + gj[mm]);
              }
              ec_flux(d, g, &P.ub[(size_t)i * Nc], &P.ub[(size_t)j * Nc], nv, F);
              out.vp++;
              for (int c = 0; c < Nc; ++c) {
                res[(size_t)i * Nc + c] -= F[c];
                res[(size_t)j * Nc + c] += F[c];
              }
            }
    }
    // ---- facet correction C (P:525 [eq:facet_correction]) ----
    vector<double> Ct1((size_t)Nf * Nqf * Nc, 0.0);
    for (int z = 0; z < Nf; ++z) {
      double rbmax = 0.0;
      for (int f = 0; f < Nqf; ++f)
        for (int i = 0; i < Nq; ++i)
          rbmax = std::max(rbmax, std::fabs(r.R[((size_t)z * Nqf + f) * Nq + i] * r.B[z * Nqf + f]));
      for (int i = 0; i < Nq; ++i)
        for (int f = 0; f < Nqf; ++f) {
          double rb = r.R[((size_t)z * Nqf + f) * Nq + i] * r.B[z * Nqf + f];  // (R^T B)_if
          if (variant != 2 && !(std::fabs(rb) > 1e-12 * rbmax)) continue;
          const double* Gfj = &m.Gf[e][((size_t)z * Nqf + f) * d * d];
          for (int mm = 0; mm < d; ++mm) {  // <J n>_ij = (G_i^T nhat + G_fj^T nhat)/2
            double s = 0.0;
            for (int l = 0; l < d; ++l) s += (G[((size_t)i * d + l) * d + mm] + Gfj[l * d + mm]) * r.nhat[z * d + l];
            nv[mm] = 0.5 * s;
          }
          ec_flux(d, g, &P.ub[(size_t)i * Nc], &P.ubf[((size_t)z * Nqf + f) * Nc], nv, F);
          out.fp++;
          for (int c = 0; c < Nc; ++c) {
            res[(size_t)i * Nc + c] -= rb * F[c];              // - C 1
            Ct1[((size_t)z * Nqf + f) * Nc + c] += rb * F[c];  // C^T 1
          }
        }
    }
    // ---- interface flux and lifting: r -= R^T (B J_f f* - C^T 1) (P:520 second line) ----
    for (int z = 0; z < Nf; ++z) {
      int64_t o = m.nbr[e * Nf + z];
      int zo = m.nbr_face[e * Nf + z], rf = m.reflect[e * Nf + z];
      const Proj& PO = PJ[slot[o]];
      for (int f = 0; f < Nqf; ++f) {
        int i1 = f % n, i2 = f / n;
        int fo = (d == 2) ? (rf ? n - 1 - f : f) : ((rf ? n - 1 - i1 : i1) + n * i2);
        const double* um = &P.ubf[((size_t)z * Nqf + f) * Nc];
        const double* up = &PO.ubf[((size_t)zo * Nqf + fo) * Nc];
        const double* Jn = &m.Jn[e][((size_t)z * Nqf + f) * d];
        double Jf = 0.0;
        for (int k = 0; k < d; ++k) Jf += Jn[k] * Jn[k];
        Jf = std::sqrt(Jf);  // P:361 [eq:nanson]
        double nu[3];
        for (int k = 0; k < d; ++k) nu[k] = Jn[k] / Jf;
        double fs[5];
        iface_flux(flux_mode, d, g, um, up, nu, fs);  // P:491 (ES), P:841 (EC), P:497 (R27)
        out.ie++;
        double bf = r.B[z * Nqf + f];
        for (int c = 0; c < Nc; ++c) {
          double sv = bf * Jf * fs[c] - Ct1[((size_t)z * Nqf + f) * Nc + c];
          for (int i = 0; i < Nq; ++i) res[(size_t)i * Nc + c] -= r.R[((size_t)z * Nqf + f) * Nq + i] * sv;
        }
      }
    }
  }
  // ---- monitors: sum w.r, sum r ----
  for (int i = 0; i < Nq; ++i)
    for (int c = 0; c < Nc; ++c) {
      double wr = P.w[(size_t)i * Nc + c] * res[(size_t)i * Nc + c];
      out.erate += wr;
      out.eabs += std::fabs(wr);
      out.cons[c] += res[(size_t)i * Nc + c];
    }
  // ---- dudt = M~^{-1} V^T r (P:593 [eq:matvec_dudt]) ----
  vector<double> rc(Nq);
  for (int c = 0; c < Nc; ++c) {
    for (int i = 0; i < Nq; ++i) rc[i] = res[(size_t)i * Nc + c];
    wadg(m, e, rc.data(), dudt + (size_t)c * r.Np);
  }
  out.ser += tl_series - s0;
  out.lg += tl_log - l0;
}

}  // namespace

extern "C" {

int ora_rhs(const ora_mesh* m, const double* u_modal, double* dudt, int flux_mode, int variant,
            int64_t n_out, const int64_t* out_elems, int nthreads, ora_stats* stats) {
  const Ref& r = m->ref;
  int Nf = r.Nf, Nc = m->Nc, Np = r.Np;
  int64_t ne = m->ne;
  vector<int64_t> outl;
  if (out_elems)
    outl.assign(out_elems, out_elems + n_out);
  else
    for (int64_t e = 0; e < ne; ++e) outl.push_back(e);
  // elements whose projection is needed: outputs and their neighbours
  vector<int64_t> slot(ne, -1), plist;
  for (int64_t e : outl) {
    if (!m->has_geom[e]) return -1;
    if (slot[e] < 0) {
      slot[e] = plist.size();
      plist.push_back(e);
    }
    for (int z = 0; z < Nf; ++z) {
      int64_t o = m->nbr[e * Nf + z];
      if (slot[o] < 0) {
        slot[o] = plist.size();
        plist.push_back(o);
      }
    }
  }
#ifdef _OPENMP
  int nt = nthreads > 0 ? nthreads : omp_get_max_threads();
#else
  int nt = 1;
  (void)nthreads;
#endif
  vector<Proj> PJ(plist.size());
  vector<int64_t> ser(plist.size(), 0), lgb(plist.size(), 0);
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int64_t a = 0; a < (int64_t)plist.size(); ++a) {
    int64_t s0 = tl_series, l0 = tl_log;
    PJ[a] = project(*m, plist[a], u_modal + (size_t)plist[a] * Nc * Np);
    ser[a] = tl_series - s0;
    lgb[a] = tl_log - l0;
  }
  for (auto& pj : PJ)
    if (!pj.admissible) {
      if (stats) {
        std::memset(stats, 0, sizeof(ora_stats));
        stats->inadmissible = 1;
      }
      return 3;
    }
  vector<ElemOut> eo(outl.size());
#pragma omp parallel for schedule(dynamic, 1) num_threads(nt)
  for (int64_t a = 0; a < (int64_t)outl.size(); ++a)
    element_rhs(*m, outl[a], PJ, slot, flux_mode, variant, dudt + (size_t)outl[a] * Nc * Np, eo[a]);
  if (stats) {
    std::memset(stats, 0, sizeof(ora_stats));
    for (auto& o : eo) {  // fixed-order reduction
      stats->volume_pairs += o.vp;
      stats->facet_pairs += o.fp;
      stats->interface_evals += o.ie;
      stats->series_branch += o.ser;
      stats->log_branch += o.lg;
      stats->entropy_rate += o.erate;
      stats->entropy_abs += o.eabs;
      for (int c = 0; c < Nc; ++c) stats->conservation[c] += o.cons[c];
    }
    stats->n_elements = (int64_t)outl.size();
  }
  return 0;
}

// ---- linear advection, du/dt + div(a u) = 0: the skew-symmetric weak form
// P:431-436 [eq:rhs_skew], or the conservative form P:425-426 [eq:rhs_cons], with dense operators ----
//   r = 1/2 sum_l ( Q^(l)T sum_m G^(l,m) f^(m) - sum_m G^(l,m) Q^(l) f^(m) )
//       - sum_z R^(z)T B^(z) J^(z) ( f* - 1/2 sum_m N^(z,m) R^(z) f^(m) ),   f^(m) = a_m u   (skew)
//   r = sum_l Q^(l)T sum_m G^(l,m) f^(m) - sum_z R^(z)T B^(z) J^(z) f*                          (conservative)
// f* = (a.n) (u- + u+)/2 (central, flux_mode 0) or minus |a.n| (u+ - u-)/2 (upwind, flux_mode 1),
// n the unit outward normal J n / J_f; d u~/dt = M~^{-1} V^T r.  energy[0] = sum_k u^T r
// = d/dt sum_k u~^T M~ u~ / 2, energy[1] = sum_k |u_i r_i|.
int ora_advection_rhs(const ora_mesh* m, const double* u_modal /*[ne][Np]*/, const double* a, int flux_mode,
                      int form, double* dudt, double* energy) {
  const Ref& r = m->ref;
  const int d = m->d, Nq = r.Nq, Np = r.Np, Nf = r.Nf, Nqf = r.Nqf, n = r.n;
  const int64_t ne = m->ne;
  for (int64_t e = 0; e < ne; ++e)
    if (!m->has_geom[e]) return -1;
  // nodal values u = V u~ and traces R^(z) u at every facet node
  vector<double> un((size_t)ne * Nq), ut((size_t)ne * Nf * Nqf);
  for (int64_t e = 0; e < ne; ++e) {
    Vapply(r, u_modal + (size_t)e * Np, &un[(size_t)e * Nq]);
    for (int z = 0; z < Nf; ++z)
      for (int f = 0; f < Nqf; ++f) {
        double t = 0.0;
        for (int i = 0; i < Nq; ++i) t += r.R[((size_t)z * Nqf + f) * Nq + i] * un[(size_t)e * Nq + i];
        ut[((size_t)e * Nf + z) * Nqf + f] = t;
      }
  }
  double er = 0.0, ea = 0.0;
  vector<double> res(Nq), c((size_t)d * Nq);
  for (int64_t e = 0; e < ne; ++e) {
    const double* u = &un[(size_t)e * Nq];
    const vector<double>& G = m->G[e];
    for (int l = 0; l < d; ++l)  // c_l = sum_m G_lm a_m, so that sum_m G^(l,m) f^(m) = c_l u
      for (int i = 0; i < Nq; ++i) {
        double t = 0.0;
        for (int mm = 0; mm < d; ++mm) t += G[((size_t)i * d + l) * d + mm] * a[mm];
        c[(size_t)l * Nq + i] = t;
      }
    for (int i = 0; i < Nq; ++i) {
      double t = 0.0;
      for (int l = 0; l < d; ++l) {
        const double* Q = &r.Q[(size_t)l * Nq * Nq];
        const double* cl = &c[(size_t)l * Nq];
        for (int j = 0; j < Nq; ++j) {
          const double qt = Q[(size_t)j * Nq + i] * cl[j] * u[j];  // (Q^T (c u))_i
          t += form == 0 ? 0.5 * (qt - cl[i] * Q[(size_t)i * Nq + j] * u[j]) : qt;
        }
      }
      res[i] = t;
    }
    for (int z = 0; z < Nf; ++z) {
      const int64_t o = m->nbr[e * Nf + z];
      const int zo = m->nbr_face[e * Nf + z], rf = m->reflect[e * Nf + z];
      for (int f = 0; f < Nqf; ++f) {
        const int i1 = f % n, i2 = f / n;
        const int fo = (d == 2) ? (rf ? n - 1 - f : f) : ((rf ? n - 1 - i1 : i1) + n * i2);
        const double um = ut[((size_t)e * Nf + z) * Nqf + f], up = ut[((size_t)o * Nf + zo) * Nqf + fo];
        const double* Jn = &m->Jn[e][((size_t)z * Nqf + f) * d];
        double Jf = 0.0, an = 0.0;
        for (int k = 0; k < d; ++k) Jf += Jn[k] * Jn[k];
        Jf = std::sqrt(Jf);
        for (int k = 0; k < d; ++k) an += a[k] * Jn[k] / Jf;
        double fs = an * 0.5 * (um + up);
        if (flux_mode == 1) fs -= 0.5 * std::fabs(an) * (up - um);
        const double sv = r.B[z * Nqf + f] * Jf * (form == 0 ? fs - 0.5 * an * um : fs);
        for (int i = 0; i < Nq; ++i) res[i] -= r.R[((size_t)z * Nqf + f) * Nq + i] * sv;
      }
    }
    for (int i = 0; i < Nq; ++i) {
      er += u[i] * res[i];
      ea += std::fabs(u[i] * res[i]);
    }
    wadg(*m, e, res.data(), dudt + (size_t)e * Np);
  }
  if (energy) {
    energy[0] = er;
    energy[1] = ea;
  }
  return 0;
}

// Dormand-Prince 5(4) (Hairer, Norsett & Wanner I, Table II.5.2; the paper integrates with DP8 of
// the same family): c, a (lower triangle, row-major 7x7), b (5th order), bh (embedded 4th)
static const double DP_C[7] = {0.0, 1.0 / 5.0, 3.0 / 10.0, 4.0 / 5.0, 8.0 / 9.0, 1.0, 1.0};
static const double DP_A[7][7] = {
    {0, 0, 0, 0, 0, 0, 0},
    {1.0 / 5.0, 0, 0, 0, 0, 0, 0},
    {3.0 / 40.0, 9.0 / 40.0, 0, 0, 0, 0, 0},
    {44.0 / 45.0, -56.0 / 15.0, 32.0 / 9.0, 0, 0, 0, 0},
    {19372.0 / 6561.0, -25360.0 / 2187.0, 64448.0 / 6561.0, -212.0 / 729.0, 0, 0, 0},
    {9017.0 / 3168.0, -355.0 / 33.0, 46732.0 / 5247.0, 49.0 / 176.0, -5103.0 / 18656.0, 0, 0},
    {35.0 / 384.0, 0.0, 500.0 / 1113.0, 125.0 / 192.0, -2187.0 / 6784.0, 11.0 / 84.0, 0}};
static const double DP_B[7] = {35.0 / 384.0, 0.0, 500.0 / 1113.0, 125.0 / 192.0, -2187.0 / 6784.0, 11.0 / 84.0, 0.0};
static const double DP_BH[7] = {5179.0 / 57600.0, 0.0, 7571.0 / 16695.0, 393.0 / 640.0, -92097.0 / 339200.0,
                                187.0 / 2100.0, 1.0 / 40.0};

void ora_dp54_tableau(double* c, double* a, double* b, double* bh) {
  for (int i = 0; i < 7; ++i) {
    c[i] = DP_C[i];
    b[i] = DP_B[i];
    bh[i] = DP_BH[i];
    for (int j = 0; j < 7; ++j) a[i * 7 + j] = DP_A[i][j];
  }
}

// one Dormand-Prince 5(4) step of size dt from u (not modified): u5 = 5th-order solution, *err =
// sqrt(mean_i (e_i / (atol + rtol max(|u_i|, |u5_i|)))^2) with e_i = dt sum_j (b_j - bh_j) k_j
// (Hairer-Norsett-Wanner I, eq. II.4.11), k_7 = f(u5) (first same as last)
int ora_dp54(const ora_mesh* m, const double* u, double dt, double rtol, double atol, int flux_mode,
             int nthreads, double* u5, double* err) {
  size_t N = (size_t)m->ne * m->Nc * m->ref.Np;
  vector<vector<double>> k(7, vector<double>(N));
  vector<double> us(N);
  int rc;
  for (int st = 0; st < 7; ++st) {
    for (size_t i = 0; i < N; ++i) {
      double s = 0.0;
      for (int j = 0; j < st; ++j) s += DP_A[st][j] * k[j][i];
      us[i] = u[i] + dt * s;
    }
    if ((rc = ora_rhs(m, us.data(), k[st].data(), flux_mode, 1, 0, nullptr, nthreads, nullptr))) return rc;
  }
  // the last stage input is the 5th-order solution (a_7j = b_j)
  double sq = 0.0;
  for (size_t i = 0; i < N; ++i) {
    u5[i] = us[i];
    double e = 0.0;
    for (int j = 0; j < 7; ++j) e += (DP_B[j] - DP_BH[j]) * k[j][i];
    e *= dt;
    double sc = atol + rtol * std::max(std::fabs(u[i]), std::fabs(u5[i]));
    sq += (e / sc) * (e / sc);
  }
  *err = std::sqrt(sq / (double)N);
  return 0;
}

int ora_rk4(const ora_mesh* m, double* u, double dt, int nsteps, int flux_mode, int nthreads) {
  // classical four-stage Runge-Kutta (R17)
  size_t N = (size_t)m->ne * m->Nc * m->ref.Np;
  vector<double> k1(N), k2(N), k3(N), k4(N), us(N);
  for (int s = 0; s < nsteps; ++s) {
    int rc;
    if ((rc = ora_rhs(m, u, k1.data(), flux_mode, 1, 0, nullptr, nthreads, nullptr))) return rc;
    for (size_t i = 0; i < N; ++i) us[i] = u[i] + 0.5 * dt * k1[i];
    if ((rc = ora_rhs(m, us.data(), k2.data(), flux_mode, 1, 0, nullptr, nthreads, nullptr))) return rc;
    for (size_t i = 0; i < N; ++i) us[i] = u[i] + 0.5 * dt * k2[i];
    if ((rc = ora_rhs(m, us.data(), k3.data(), flux_mode, 1, 0, nullptr, nthreads, nullptr))) return rc;
    for (size_t i = 0; i < N; ++i) us[i] = u[i] + dt * k3[i];
    if ((rc = ora_rhs(m, us.data(), k4.data(), flux_mode, 1, 0, nullptr, nthreads, nullptr))) return rc;
    for (size_t i = 0; i < N; ++i) u[i] += dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  }
  return 0;
}

}  // extern "C"
