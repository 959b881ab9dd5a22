// tables.cpp -- host construction of the reference tables used by the sm_100a kernels.
//
// Independent of oracle/: nodes by Golub-Welsch (implicit-QL eigenvalues of the Jacobi matrix)
// polished by Newton on the monic recurrence, weights by the Gauss-Christoffel formula, Lagrange
// data by the barycentric formula, and PKD gradients by forward-mode dual numbers.
// Citations: P:<line> = PAPER.md.
#include <quadmath.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cmath>
#include <cstring>

#include "internal.h"

namespace esb {
namespace {

typedef __float128 Q;  // every table is evaluated in binary128 and rounded once (R26)
inline Q qsqrt(Q x) { return sqrtq(x); }

// ---------------- monic Jacobi recurrence p_{k+1} = (x - al_k) p_k - be_k p_{k-1} ----------------
struct Monic {
  std::vector<double> al, be;  // be[0] = mu0 = int (1-x)^a (1+x)^b
};
Monic monic_coeffs(int N, double a, double b) {
  Monic m;
  m.al.resize(N + 1);
  m.be.resize(N + 1);
  for (int k = 0; k <= N; ++k) {
    double s = 2.0 * k + a + b;
    m.al[k] = (k == 0) ? (b - a) / (a + b + 2.0) : (b * b - a * a) / (s * (s + 2.0));
    if (k == 0)
      m.be[k] = std::exp((a + b + 1.0) * std::log(2.0) + std::lgamma(a + 1.0) + std::lgamma(b + 1.0) -
                         std::lgamma(a + b + 2.0));
    else if (k == 1)
      m.be[k] = 4.0 * (1.0 + a) * (1.0 + b) / ((2.0 + a + b) * (2.0 + a + b) * (3.0 + a + b));
    else
      m.be[k] = 4.0 * k * (k + a) * (k + b) * (k + a + b) / (s * s * (s + 1.0) * (s - 1.0));
  }
  return m;
}

// normalised Jacobi value via the orthonormal recurrence derived from the monic one
double pnorm(int n, double a, double b, double x) {
  Monic m = monic_coeffs(n + 1, a, b);
  double pm = 0.0, pc = 1.0 / sqrt(m.be[0]);
  for (int k = 0; k < n; ++k) {
    double pn = ((x - m.al[k]) * pc - (k > 0 ? sqrt(m.be[k]) * pm : 0.0)) / sqrt(m.be[k + 1]);
    pm = pc;
    pc = pn;
  }
  return pc;
}

struct MonicQ {
  std::vector<Q> al, be;
};
MonicQ monic_q(int N, Q a, Q b) {
  MonicQ m;
  m.al.resize(N + 1);
  m.be.resize(N + 1);
  for (int k = 0; k <= N; ++k) {
    Q s = (Q)2 * k + a + b;
    m.al[k] = (k == 0) ? (b - a) / (a + b + (Q)2) : (b * b - a * a) / (s * (s + (Q)2));
    if (k == 0)
      m.be[k] = expq((a + b + (Q)1) * logq((Q)2) + lgammaq(a + (Q)1) + lgammaq(b + (Q)1) - lgammaq(a + b + (Q)2));
    else if (k == 1)
      m.be[k] = (Q)4 * ((Q)1 + a) * ((Q)1 + b) / (((Q)2 + a + b) * ((Q)2 + a + b) * ((Q)3 + a + b));
    else
      m.be[k] = (Q)4 * k * (k + a) * (k + b) * (k + a + b) / (s * s * (s + (Q)1) * (s - (Q)1));
  }
  return m;
}
// normalised Jacobi value in binary128
Q pnorm_q(int n, Q a, Q b, Q x) {
  MonicQ m = monic_q(n + 1, a, b);
  Q pm = 0, pc = (Q)1 / qsqrt(m.be[0]);
  for (int k = 0; k < n; ++k) {
    Q pn = ((x - m.al[k]) * pc - (k > 0 ? qsqrt(m.be[k]) * pm : (Q)0)) / qsqrt(m.be[k + 1]);
    pm = pc;
    pc = pn;
  }
  return pc;
}

// Eigenvalues of the symmetric tridiagonal Jacobi matrix (diagonal dg, off-diagonal e) by bisection on
// the Sturm count: the number of negative pivots of the LDL^T factorisation of (J - t I) equals the
// number of eigenvalues below t.  Only the eigenvalues are needed (starting values of the binary128
// Newton polish in gauss_rule); they all lie in [-1, 1] for the Jacobi weights on [-1, 1].
int sturm_below(const std::vector<double>& dg, const std::vector<double>& e, int n, double t) {
  int cnt = 0;
  double q = 1.0;
  for (int k = 0; k < n; ++k) {
    q = dg[k] - t - (k > 0 ? e[k - 1] * e[k - 1] / q : 0.0);
    if (q == 0.0) q = -1e-300;
    if (q < 0.0) ++cnt;
  }
  return cnt;
}
bool tridiag_eigvals(const std::vector<double>& dg, const std::vector<double>& e, int n, std::vector<double>& lam) {
  lam.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {  // i-th smallest eigenvalue: count(below lo) <= i < count(below hi)
    double lo = -1.0 - 1e-12, hi = 1.0 + 1e-12;
    for (int it = 0; it < 200 && hi - lo > 1e-15; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (sturm_below(dg, e, n, mid) > i)
        hi = mid;
      else
        lo = mid;
    }
    lam[i] = 0.5 * (lo + hi);
  }
  return true;
}

// Gauss rule w.r.t. (1-x)^a (1+x)^b with N nodes: the eigenvalues of the Jacobi matrix
// (Golub-Welsch) by Sturm bisection as starting values, Newton on the monic recurrence in binary128, Gauss-Christoffel weights
//   w_i = ||p_{N-1}||^2 / (p_{N-1}(x_i) p_N'(x_i)).
bool gauss_rule(int N, double a, double b, std::vector<Q>& x, std::vector<Q>& w) {
  Monic m = monic_coeffs(N + 1, a, b);
  std::vector<double> dg(N), e(N, 0.0), lam;
  for (int k = 0; k < N; ++k) dg[k] = m.al[k];
  for (int k = 0; k + 1 < N; ++k) e[k] = std::sqrt(m.be[k + 1]);
  if (!tridiag_eigvals(dg, e, N, lam)) return false;
  dg = lam;
  MonicQ mq = monic_q(N + 1, a, b);
  Q norm2 = mq.be[0];
  for (int k = 1; k < N; ++k) norm2 *= mq.be[k];
  x.resize(N);
  w.resize(N);
  for (int i = 0; i < N; ++i) {
    Q xi = dg[i];
    Q pN = 0, dpN = 0, pN1 = 0;
    for (int it = 0; it < 6; ++it) {
      Q p0 = 1, d0 = 0, p1 = xi - mq.al[0], d1 = 1;
      for (int k = 1; k < N; ++k) {
        Q p2 = (xi - mq.al[k]) * p1 - mq.be[k] * p0;
        Q d2 = p1 + (xi - mq.al[k]) * d1 - mq.be[k] * d0;
        p0 = p1;
        d0 = d1;
        p1 = p2;
        d1 = d2;
      }
      pN = p1;
      dpN = d1;
      pN1 = p0;
      if (it < 5) xi -= pN / dpN;
    }
    x[i] = xi;
    w[i] = norm2 / (pN1 * dpN);
  }
  return true;
}

// barycentric Lagrange data on nodes x (binary128)
std::vector<Q> bary_weights(const std::vector<Q>& x) {
  int n = (int)x.size();
  std::vector<Q> lam(n, (Q)1);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k)
      if (k != j) lam[j] /= (x[j] - x[k]);
  return lam;
}
std::vector<Q> lagrange_at(const std::vector<Q>& x, Q t) {
  int n = (int)x.size();
  std::vector<Q> lam = bary_weights(x), l(n, (Q)0);
  for (int j = 0; j < n; ++j)
    if (t == x[j]) {
      l[j] = 1;
      return l;
    }
  Q den = 0;
  for (int j = 0; j < n; ++j) den += lam[j] / (t - x[j]);
  for (int j = 0; j < n; ++j) l[j] = lam[j] / (t - x[j]) / den;
  return l;
}
std::vector<Q> diff_matrix(const std::vector<Q>& x) {  // D[i][j] = l_j'(x_i)
  int n = (int)x.size();
  std::vector<Q> lam = bary_weights(x), D((size_t)n * n, (Q)0);
  for (int i = 0; i < n; ++i) {
    Q s = 0;
    for (int j = 0; j < n; ++j)
      if (j != i) {
        D[(size_t)i * n + j] = lam[j] / lam[i] / (x[i] - x[j]);
        s += D[(size_t)i * n + j];
      }
    D[(size_t)i * n + i] = -s;
  }
  return D;
}
std::vector<double> skew_of(const std::vector<Q>& X, int n) {
  std::vector<double> S((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) S[(size_t)i * n + j] = (double)((X[(size_t)i * n + j] - X[(size_t)j * n + i]) / (Q)2);
  return S;
}
std::vector<double> rnd(const std::vector<Q>& v) {
  std::vector<double> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = (double)v[i];
  return o;
}

// ---------------- geometry tables in binary128 ----------------
// The geometry of an element is built from Lagrange interpolants on the equispaced barycentric
// lattice of degree N (R10).  For that lattice the Lagrange basis has Silvester's closed form
//   l_alpha(lam) = prod_k prod_{j < alpha_k} (N lam_k - j) / (j + 1),   |alpha| = N,
// so the tables need no Vandermonde inverse.  They are evaluated in binary128 and stored as
// double-double pairs because the device sums them against data with cancellation (R25).
typedef __float128 LD;
// equispaced barycentric lattice of degree N (R10): reference coords [M][d], barycentric [M][d+1]
template <class T>
void lattice_nodes(int d, int N, std::vector<T>& xi, std::vector<double>& bary) {
  xi.clear();
  bary.clear();
  if (d == 2) {
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j) {
        double l2 = double(i) / N, l3 = double(j) / N;
        bary.insert(bary.end(), {1.0 - l2 - l3, l2, l3});
        xi.insert(xi.end(), {(T)(2 * i) / N - 1, (T)(2 * j) / N - 1});
      }
  } else {
    for (int i = 0; i <= N; ++i)
      for (int j = 0; j <= N - i; ++j)
        for (int k = 0; k <= N - i - j; ++k) {
          double l2 = double(i) / N, l3 = double(j) / N, l4 = double(k) / N;
          bary.insert(bary.end(), {1.0 - l2 - l3 - l4, l2, l3, l4});
          xi.insert(xi.end(), {(T)(2 * i) / N - 1, (T)(2 * j) / N - 1, (T)(2 * k) / N - 1});
        }
  }
}

// Lagrange basis (and gradients) of the degree-N lattice evaluated at points X[npts][d] (reference
// coordinates, binary128): Lq [npts][M], Dq [d][npts][M]
void lattice_basis_q(int d, int N, const std::vector<LD>& X, int npts, std::vector<LD>* Lq, std::vector<LD>* Dq) {
  std::vector<double> lxi, lb;
  lattice_nodes<double>(d, N, lxi, lb);
  const int nb = d + 1, M = (int)lb.size() / nb;
  std::vector<int> alpha((size_t)M * nb);
  for (int i = 0; i < M; ++i)
    for (int k = 0; k < nb; ++k) alpha[(size_t)i * nb + k] = (int)std::lround(lb[(size_t)i * nb + k] * N);
  if (Lq) Lq->assign((size_t)npts * M, (LD)0);
  if (Dq) Dq->assign((size_t)d * npts * M, (LD)0);
#pragma omp parallel for schedule(dynamic, 8)
  for (int x = 0; x < npts; ++x) {
    // barycentric coordinates: lam_{k+1} = (1 + xi_k)/2, lam_1 = 1 - sum; d lam_{k+1}/d xi_l = delta/2,
    // d lam_1 / d xi_l = -1/2
    LD lam[4];
    LD sum = 0;
    for (int k = 0; k < d; ++k) {
      lam[k + 1] = ((LD)1 + X[(size_t)x * d + k]) / (LD)2;
      sum += lam[k + 1];
    }
    lam[0] = (LD)1 - sum;
    for (int i = 0; i < M; ++i) {
      const int* al = &alpha[(size_t)i * nb];
      LD f[4], df[4];  // factor prod_{j<a}(N lam - j)/(j+1) and its derivative w.r.t. lam
      for (int k = 0; k < nb; ++k) {
        LD v = 1, dv = 0;
        for (int j = 0; j < al[k]; ++j) {
          LD t = ((LD)N * lam[k] - (LD)j) / (LD)(j + 1);
          dv = dv * t + v * (LD)N / (LD)(j + 1);
          v = v * t;
        }
        f[k] = v;
        df[k] = dv;
      }
      LD val = 1;
      for (int k = 0; k < nb; ++k) val *= f[k];
      if (Lq) (*Lq)[(size_t)x * M + i] = val;
      if (Dq) {
        for (int l = 0; l < d; ++l) {
          // d/dxi_l = 1/2 (d/dlam_{l+1} - d/dlam_0)
          LD g = 0;
          for (int k = 0; k < nb; ++k) {
            if (k != l + 1 && k != 0) continue;
            LD prod = df[k];
            for (int kk = 0; kk < nb; ++kk)
              if (kk != k) prod *= f[kk];
            g += (k == 0) ? -prod : prod;
          }
          (*Dq)[((size_t)l * npts + x) * M + i] = g / (LD)2;
        }
      }
    }
  }
}

// ---------------- warp & blend node family (reading R32) ----------------
// Warburton's warp & blend with the blending parameter alpha = 0, in barycentric form.  1D warp
// factor wf(r) = w(r) / (1 - r^2), w the degree-N interpolant (barycentric Lagrange formula) on the
// equispaced points of their displacement to the Gauss-Lobatto-Legendre points -- whose interior
// points are the nodes of the Gauss-Jacobi (1,1) rule.  A triangle with barycentrics lam moves by
// sum over its edges (u, v) of 2 lam_u lam_v wf(lam_v - lam_u) (e_v - e_u) (the edge warp blended by
// 4 lam_u lam_v); a tetrahedron by the sum over its faces of the face's triangle warp (in the raw
// barycentrics of its three vertices) times lam_b lam_c lam_d / prod(lam_x + lam_a / 2), a the opposite
// vertex, except on edges, which take the face warp itself.  Nodes in lattice_nodes order.
void node_bary(int d, int N, int family, std::vector<LD>& bary) {
  std::vector<double> xi, b;
  lattice_nodes<double>(d, N, xi, b);
  const int nb = d + 1, M = (int)b.size() / nb;
  bary.assign(b.size(), (LD)0);
  for (int i = 0; i < M; ++i) {
    LD s = 0;
    for (int k = 1; k < nb; ++k) {
      bary[(size_t)i * nb + k] = (LD)std::lround(b[(size_t)i * nb + k] * N) / (LD)N;
      s += bary[(size_t)i * nb + k];
    }
    bary[(size_t)i * nb] = (LD)1 - s;
  }
  if (family != 1 || N < 3) return;  // N <= 2: the GLL points are equispaced
  std::vector<LD> gx, gw, req(N + 1), disp(N + 1);
  gauss_rule(N - 1, 1.0, 1.0, gx, gw);
  std::sort(gx.begin(), gx.end());
  for (int i = 0; i <= N; ++i) {
    req[i] = (LD)(2 * i - N) / (LD)N;
    const LD g = i == 0 ? (LD)-1 : (i == N ? (LD)1 : gx[i - 1]);
    disp[i] = g - req[i];
  }
  auto wf = [&](LD r) -> LD {
    const LD ar = r < 0 ? -r : r;
    if (ar >= (LD)1 - (LD)1e-24) return 0;
    const std::vector<LD> l = lagrange_at(req, r);
    LD w = 0;
    for (int i = 0; i <= N; ++i) w += disp[i] * l[i];
    return w / ((LD)1 - r * r);
  };
  const LD tol = (LD)1e-10;
  for (int i = 0; i < M; ++i) {
    LD* L = &bary[(size_t)i * nb];
    LD sh[4] = {0, 0, 0, 0};
    auto tri_warp = [&](int a, int b2, int c, LD* W) {
      for (int k = 0; k < 4; ++k) W[k] = 0;
      const int ed[3][2] = {{a, b2}, {b2, c}, {a, c}};
      for (const auto& e : ed) {
        const LD t = 2 * L[e[0]] * L[e[1]] * wf(L[e[1]] - L[e[0]]);
        W[e[1]] += t;
        W[e[0]] -= t;
      }
    };
    if (d == 2) {
      tri_warp(0, 1, 2, sh);
    } else {
      for (int o = 0; o < 4; ++o) {
        int v[3], q = 0;
        for (int k = 0; k < 4; ++k)
          if (k != o) v[q++] = k;
        LD W[4];
        tri_warp(v[0], v[1], v[2], W);
        const LD la = L[o], half = la / 2;
        LD blend = L[v[0]] * L[v[1]] * L[v[2]];
        const LD den = (L[v[0]] + half) * (L[v[1]] + half) * (L[v[2]] + half);
        if (den > tol) blend /= den;
        const int inside = (L[v[0]] > tol) + (L[v[1]] > tol) + (L[v[2]] > tol);
        for (int k = 0; k < 4; ++k) sh[k] = (la < tol && inside < 3) ? W[k] : sh[k] + blend * W[k];
      }
    }
    for (int k = 0; k < nb; ++k) L[k] += sh[k];
  }
}

// inverse of a dense M x M matrix in binary128 (Gauss-Jordan, partial pivoting)
bool invert_q(std::vector<LD>& A, int M) {
  std::vector<LD> I((size_t)M * M, (LD)0);
  for (int i = 0; i < M; ++i) I[(size_t)i * M + i] = 1;
  for (int c = 0; c < M; ++c) {
    int pr = c;
    for (int r = c + 1; r < M; ++r)
      if (fabsq(A[(size_t)r * M + c]) > fabsq(A[(size_t)pr * M + c])) pr = r;
    if (A[(size_t)pr * M + c] == 0) return false;
    if (pr != c)
      for (int k = 0; k < M; ++k) {
        std::swap(A[(size_t)pr * M + k], A[(size_t)c * M + k]);
        std::swap(I[(size_t)pr * M + k], I[(size_t)c * M + k]);
      }
    const LD iv = (LD)1 / A[(size_t)c * M + c];
    for (int k = 0; k < M; ++k) {
      A[(size_t)c * M + k] *= iv;
      I[(size_t)c * M + k] *= iv;
    }
    for (int r = 0; r < M; ++r) {
      if (r == c) continue;
      const LD f = A[(size_t)r * M + c];
      if (f == 0) continue;
      for (int k = 0; k < M; ++k) {
        A[(size_t)r * M + k] -= f * A[(size_t)c * M + k];
        I[(size_t)r * M + k] -= f * I[(size_t)c * M + k];
      }
    }
  }
  A.swap(I);
  return true;
}

// Lagrange basis (and gradients) of the degree-N node family at points X[npts][d] (binary128), stored
// as double-double pairs: out = [hi block | lo block].  Family 0: the lattice's closed form.  Family 1
// (warp & blend): l^wb(x) = l^lat(x) A^-1 with A_ij = l^lat_j(x^wb_i), A^-1 cached per (d, N).
bool node_basis(int d, int N, int family, const std::vector<LD>& X, int npts, std::vector<double>* L,
                std::vector<double>* Dg /*[d][npts][M]*/) {
  std::vector<LD> Lq, Dq;
  lattice_basis_q(d, N, X, npts, L ? &Lq : nullptr, Dg ? &Dq : nullptr);
  const int M = d == 2 ? (N + 1) * (N + 2) / 2 : (N + 1) * (N + 2) * (N + 3) / 6;
  if (family == 1 && N >= 3) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, std::vector<LD>> cache;
    std::vector<LD> Ai;
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = cache.find({d, N});
      if (it == cache.end()) {
        std::vector<LD> bw, xw((size_t)M * d), A;
        node_bary(d, N, 1, bw);
        for (int i = 0; i < M; ++i)
          for (int k = 0; k < d; ++k) xw[(size_t)i * d + k] = 2 * bw[(size_t)i * (d + 1) + k + 1] - 1;
        lattice_basis_q(d, N, xw, M, &A, nullptr);
        if (!invert_q(A, M)) A.clear();
        it = cache.emplace(std::make_pair(d, N), A).first;
      }
      Ai = it->second;
    }
    if (Ai.empty()) return false;  // singular (not for N <= 11: the family is unisolvent)
    auto apply = [&](std::vector<LD>& B, int rows) {  // B [rows][M] <- B A^-1
      std::vector<LD> out((size_t)rows * M, (LD)0);
#pragma omp parallel for schedule(static)
      for (int r = 0; r < rows; ++r)
        for (int j = 0; j < M; ++j) {
          const LD b = B[(size_t)r * M + j];
          if (b == 0) continue;
          for (int k = 0; k < M; ++k) out[(size_t)r * M + k] += b * Ai[(size_t)j * M + k];
        }
      B.swap(out);
    };
    if (L) apply(Lq, npts);
    if (Dg) apply(Dq, d * npts);
  }
  auto pack = [](const std::vector<LD>& q, std::vector<double>& out) {
    const size_t n = q.size();
    out.assign(2 * n, 0.0);
    for (size_t i = 0; i < n; ++i) {
      const double hi = (double)q[i];
      out[i] = hi;
      out[n + i] = (double)(q[i] - (LD)hi);
    }
  };
  if (L) pack(Lq, *L);
  if (Dg) pack(Dq, *Dg);
  return true;
}
std::vector<LD> to_q(const std::vector<double>& v) { return std::vector<LD>(v.begin(), v.end()); }

void collapse(int d, const double* e, double* x) {
  if (d == 2) {
    x[0] = 0.5 * (1.0 + e[0]) * (1.0 - e[1]) - 1.0;
    x[1] = e[1];
  } else {  // P:263 with the (1-eta3) factor (R1)
    x[0] = 0.25 * (1.0 + e[0]) * (1.0 - e[1]) * (1.0 - e[2]) - 1.0;
    x[1] = 0.5 * (1.0 + e[1]) * (1.0 - e[2]) - 1.0;
    x[2] = e[2];
  }
}

}  // namespace

bool build_ref_tables(int d, int p, RefTables& t, std::string& err, int nodes) {
  if (!((d == 2 && p >= 1 && p <= 10) || (d == 3 && p >= 1 && p <= 8))) {
    err = "unsupported (dim, p)";
    return false;
  }
  t.d = d;
  t.p = p;
  int n = p + 1;
  t.n = n;
  t.Nq = d == 2 ? n * n : n * n * n;
  t.Nf = d + 1;
  t.Nqf = d == 2 ? n : n * n;
  t.Np = d == 2 ? (p + 1) * (p + 2) / 2 : (p + 1) * (p + 2) * (p + 3) / 6;
  std::vector<Q> e, w, e3, w3;  // binary128 rules; rounded copies go to the device
  if (!gauss_rule(n, 0.0, 0.0, e, w) || !gauss_rule(n, 1.0, 0.0, e3, w3)) {
    err = "Gauss rule construction failed";
    return false;
  }
  t.eta = rnd(e);
  t.w = rnd(w);
  t.eta3 = rnd(e3);
  t.w3 = rnd(w3);
  // 1D line operators: X = diag(weight) D, S-line = skew(X)
  std::vector<Q> D = diff_matrix(e), D3 = diff_matrix(e3);
  std::vector<Q> Q1(n * n), A1(n * n), A2(n * n), A3(n * n), A4(n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      Q1[i * n + j] = w[i] * D[i * n + j];
      A1[i * n + j] = w[i] * ((Q)1 + e[i]) / (Q)2 * D[i * n + j];
      A2[i * n + j] = w[i] * ((Q)1 - e[i]) / (Q)2 * D[i * n + j];
      A3[i * n + j] = w[i] * ((Q)1 - e[i] * e[i]) / (Q)4 * D[i * n + j];
      A4[i * n + j] = w3[i] * ((Q)1 - e3[i]) * D3[i * n + j];
    }
  t.skQ1 = skew_of(Q1, n);
  t.skA1 = skew_of(A1, n);
  t.skA2 = skew_of(A2, n);
  t.skA3 = skew_of(A3, n);
  t.skA4 = skew_of(A4, n);
  // the full line matrices (Q^(l) restricted to a line = coefficient x X, used by the linear-advection
  // workload's skew-symmetric form P:431-436)
  t.fQ1 = rnd(Q1);
  t.fA1 = rnd(A1);
  t.fA2 = rnd(A2);
  t.fA3 = rnd(A3);
  t.fA4 = rnd(A4);
  t.lL = rnd(lagrange_at(e, (Q)-1));
  t.lR = rnd(lagrange_at(e, (Q)1));
  t.l3L = rnd(lagrange_at(e3, (Q)-1));
  t.lint4.assign(n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    std::vector<Q> l = lagrange_at(e, e3[j]);
    for (int b = 0; b < n; ++b) t.lint4[j * n + b] = (double)l[b];
  }
  // PKD principal-function tables
  t.psi1.assign(n * n, 0.0);
  t.psi2.assign((size_t)n * n * n, 0.0);
  t.psi3.assign((size_t)n * n * n, 0.0);
  for (int a1 = 0; a1 <= p; ++a1)
    for (int a = 0; a < n; ++a) t.psi1[a1 * n + a] = (double)(qsqrt((Q)2) * pnorm_q(a1, 0, 0, e[a]));
  for (int a1 = 0; a1 <= p; ++a1)
    for (int a2 = 0; a2 <= p - a1; ++a2)
      for (int b = 0; b < n; ++b)
        t.psi2[((size_t)a1 * n + a2) * n + b] =
            (double)(powq((Q)1 - e[b], (Q)a1) * pnorm_q(a2, (Q)(2 * a1 + 1), 0, e[b]));
  if (d == 3)
    for (int s = 0; s <= p; ++s)
      for (int a3 = 0; a3 <= p - s; ++a3)
        for (int c = 0; c < n; ++c)
          t.psi3[((size_t)s * n + a3) * n + c] =
              (double)((Q)2 * powq((Q)1 - e3[c], (Q)s) * pnorm_q(a3, (Q)(2 * s + 2), 0, e3[c]));
  // modal order (ABI): a1-major nested
  t.pair_a1.clear();
  t.pair_a2.clear();
  t.pair_off.clear();
  int off = 0;
  for (int a1 = 0; a1 <= p; ++a1) {
    if (d == 2) {
      t.pair_a1.push_back(a1);
      t.pair_a2.push_back(0);
      t.pair_off.push_back(off);
      off += p - a1 + 1;
    } else {
      for (int a2 = 0; a2 <= p - a1; ++a2) {
        t.pair_a1.push_back(a1);
        t.pair_a2.push_back(a2);
        t.pair_off.push_back(off);
        off += p - a1 - a2 + 1;
      }
    }
  }
  if (off != t.Np) {
    err = "modal count mismatch";
    return false;
  }
  // nodes and weights
  t.Wvol.assign(t.Nq, 0.0);
  t.xi_vol.assign((size_t)t.Nq * d, 0.0);
  t.Bf.assign((size_t)t.Nf * t.Nqf, 0.0);
  t.xi_face.assign((size_t)t.Nf * t.Nqf * d, 0.0);
  t.nhat.assign((size_t)t.Nf * 3, 0.0);
  auto collapse_q = [&](const Q* et, double* x) {  // P:183 / P:263 (R1), rounded
    if (d == 2) {
      x[0] = (double)(((Q)1 + et[0]) * ((Q)1 - et[1]) / (Q)2 - (Q)1);
      x[1] = (double)et[1];
    } else {
      x[0] = (double)(((Q)1 + et[0]) * ((Q)1 - et[1]) * ((Q)1 - et[2]) / (Q)4 - (Q)1);
      x[1] = (double)(((Q)1 + et[1]) * ((Q)1 - et[2]) / (Q)2 - (Q)1);
      x[2] = (double)et[2];
    }
  };
  if (d == 2) {
    for (int b = 0; b < n; ++b)
      for (int a = 0; a < n; ++a) {
        int i = a + n * b;
        Q et[2] = {e[a], e[b]};
        collapse_q(et, &t.xi_vol[i * 2]);
        t.Wvol[i] = (double)(w[a] * w[b] * ((Q)1 - e[b]) / (Q)2);
      }
    for (int f = 0; f < n; ++f) {
      Q f1[2] = {e[f], -1}, f2[2] = {1, e[f]}, f3[2] = {-1, e[f]};
      collapse_q(f1, &t.xi_face[(0 * n + f) * 2]);
      collapse_q(f2, &t.xi_face[(1 * n + f) * 2]);
      collapse_q(f3, &t.xi_face[(2 * n + f) * 2]);
      t.Bf[0 * n + f] = (double)w[f];
      t.Bf[1 * n + f] = (double)(qsqrt((Q)2) * w[f]);
      t.Bf[2 * n + f] = (double)w[f];
    }
    double r2 = (double)((Q)1 / qsqrt((Q)2));
    double nh[9] = {0, -1, 0, r2, r2, 0, -1, 0, 0};
    std::memcpy(t.nhat.data(), nh, sizeof(nh));
  } else {
    for (int c = 0; c < n; ++c)
      for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
          int i = a + n * b + n * n * c;
          Q et[3] = {e[a], e[b], e3[c]};
          collapse_q(et, &t.xi_vol[i * 3]);
          t.Wvol[i] = (double)(w[a] * w[b] * w3[c] * ((Q)1 - e[b]) * ((Q)1 - e3[c]) / (Q)8);
        }
    int Nqf = t.Nqf;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        int f = i + n * j;
        Q f1[3] = {e[i], -1, e3[j]}, f2[3] = {1, e[i], e3[j]}, f3[3] = {-1, e[i], e3[j]}, f4[3] = {e[i], e3[j], -1};
        collapse_q(f1, &t.xi_face[(0 * Nqf + f) * 3]);
        collapse_q(f2, &t.xi_face[(1 * Nqf + f) * 3]);
        collapse_q(f3, &t.xi_face[(2 * Nqf + f) * 3]);
        collapse_q(f4, &t.xi_face[(3 * Nqf + f) * 3]);
        Q ww = w[i] * w3[j];
        t.Bf[0 * Nqf + f] = (double)(ww / (Q)2);
        t.Bf[1 * Nqf + f] = (double)(qsqrt((Q)3) / (Q)2 * ww);
        t.Bf[2 * Nqf + f] = (double)(ww / (Q)2);
        t.Bf[3 * Nqf + f] = (double)(ww / (Q)2);
      }
    double r3 = (double)((Q)1 / qsqrt((Q)3));
    double nh[12] = {0, -1, 0, r3, r3, r3, -1, 0, 0, 0, 0, -1};
    std::memcpy(t.nhat.data(), nh, sizeof(nh));
  }
  // geometry interpolation matrices (P:327 mapping of degree p_g = p, P:349 curl interpolation of
  // degree q+1) on the node family `nodes` (0: equispaced lattice R10, 1: warp & blend R32)
  if (nodes != 0 && nodes != 1) {
    err = "mapping_nodes must be 0 or 1";
    return false;
  }
  t.nodes = nodes;
  // reference coordinates of a node family: the lattice's as before (double), warp & blend in binary128
  auto family_xi = [&](int N, std::vector<double>& bary) {
    std::vector<LD> xq;
    if (nodes == 0) {
      std::vector<double> lxi;
      lattice_nodes<double>(d, N, lxi, bary);
      xq = to_q(lxi);
    } else {
      std::vector<LD> bq;
      node_bary(d, N, 1, bq);
      bary = rnd(bq);
      const int M = (int)bq.size() / (d + 1);
      xq.resize((size_t)M * d);
      for (int i = 0; i < M; ++i)
        for (int k = 0; k < d; ++k) xq[(size_t)i * d + k] = 2 * bq[(size_t)i * (d + 1) + k + 1] - 1;
    }
    return xq;
  };
  const std::vector<LD> mxi = family_xi(p, t.lat_bary), vxi = to_q(t.xi_vol), fxi = to_q(t.xi_face);
  t.Npg = (int)t.lat_bary.size() / (d + 1);
  bool ok = node_basis(d, p, nodes, vxi, t.Nq, &t.LmapV, d == 2 ? &t.DmapV : nullptr) &&
            node_basis(d, p, nodes, mxi, t.Npg, nullptr, &t.DmapM);
  if (d == 2) {
    ok = ok && node_basis(d, p, nodes, fxi, t.Nf * t.Nqf, nullptr, &t.DmapF);
  } else {
    std::vector<double> cb;
    const std::vector<LD> cxi = family_xi(p + 1, cb);
    t.Ncl = (int)cb.size() / (d + 1);
    ok = ok && node_basis(d, p, nodes, cxi, t.Ncl, &t.LmapC, &t.DmapC) &&
         node_basis(d, p + 1, nodes, vxi, t.Nq, nullptr, &t.DcurlV) &&
         node_basis(d, p + 1, nodes, fxi, t.Nf * t.Nqf, nullptr, &t.DcurlF);
  }
  if (!ok) err = "singular node-family Vandermonde";
  return ok;
}

// Dense operators for the brute-force ablation (es_options.volume_mode = 2):
// S^(l)_ij assembled from the line operators exactly as the line-wise kernel applies them (the
// eta_k-line coefficients of DESIGN.md section 5.3), stored transposed [l][j][i]; (R^(z)T B)_if as
// [z][f][i].  Entries off the lines are zero and are evaluated anyway by the brute-force kernel.
// PKD basis (the product of the psi tables' functions, modal order of the ABI) and the
// mapping-lattice Lagrange basis with its gradients at arbitrary reference points xi[npts][d]:
// pkd [npts][Np], lmap [npts][Npg], dmap [d][npts][Npg] (rounded from binary128)
bool eval_point_tables(int d, int p, const double* xi, int npts, std::vector<double>& pkd, std::vector<double>& lmap,
                       std::vector<double>& dmap, int nodes) {
  const int Np = d == 2 ? (p + 1) * (p + 2) / 2 : (p + 1) * (p + 2) * (p + 3) / 6;
  pkd.assign((size_t)npts * Np, 0.0);
  std::vector<double> X(xi, xi + (size_t)npts * d), L, D;
  if (!node_basis(d, p, nodes, to_q(X), npts, &L, &D)) return false;
  const size_t nL = L.size() / 2, nD = D.size() / 2;
  lmap.assign(nL, 0.0);
  dmap.assign(nD, 0.0);
  for (size_t k = 0; k < nL; ++k) lmap[k] = L[k] + L[nL + k];
  for (size_t k = 0; k < nD; ++k) dmap[k] = D[k] + D[nD + k];
#pragma omp parallel for schedule(dynamic, 16)
  for (int x = 0; x < npts; ++x) {
    // collapsed coordinates (inverse of P:183 / P:263), singular vertices mapped to eta = 1
    Q e1, e2, e3 = 0;
    const double* q = xi + (size_t)x * d;
    if (d == 2) {
      e2 = q[1];
      e1 = (std::fabs(1.0 - q[1]) < 1e-300) ? (Q)1 : (Q)2 * ((Q)1 + (Q)q[0]) / ((Q)1 - (Q)q[1]) - (Q)1;
    } else {
      e3 = q[2];
      const Q den2 = (Q)1 - (Q)q[2];
      e2 = (std::fabs((double)den2) < 1e-300) ? (Q)1 : (Q)2 * ((Q)1 + (Q)q[1]) / den2 - (Q)1;
      const Q den1 = -(Q)q[1] - (Q)q[2];
      e1 = (std::fabs((double)den1) < 1e-300) ? (Q)1 : (Q)2 * ((Q)1 + (Q)q[0]) / den1 - (Q)1;
    }
    int k = 0;
    for (int a1 = 0; a1 <= p; ++a1) {
      const Q f1 = qsqrt((Q)2) * pnorm_q(a1, 0, 0, e1);
      for (int a2 = 0; a2 <= p - a1; ++a2) {
        const Q f2 = powq((Q)1 - e2, (Q)a1) * pnorm_q(a2, (Q)(2 * a1 + 1), 0, e2);
        if (d == 2) {
          pkd[(size_t)x * Np + k++] = (double)(f1 * f2);
          continue;
        }
        for (int a3 = 0; a3 <= p - a1 - a2; ++a3) {
          const int sd = a1 + a2;
          const Q f3 = (Q)2 * powq((Q)1 - e3, (Q)sd) * pnorm_q(a3, (Q)(2 * sd + 2), 0, e3);
          pkd[(size_t)x * Np + k++] = (double)(f1 * f2 * f3);
        }
      }
    }
  }
  return true;
}

void build_dense_tables(const RefTables& t, std::vector<double>& S, std::vector<double>& RB) {
  const int d = t.d, N = t.n, Nq = t.Nq, Nqf = t.Nqf, Nf = t.Nf;
  S.assign((size_t)d * Nq * Nq, 0.0);
  RB.assign((size_t)Nf * Nqf * Nq, 0.0);
  auto s_at = [&](int l, int i, int j) -> double& { return S[((size_t)l * Nq + j) * Nq + i]; };
  auto rb_at = [&](int z, int f, int i) -> double& { return RB[((size_t)z * Nqf + f) * Nq + i]; };
  if (d == 2) {
    for (int b = 0; b < N; ++b)
      for (int a = 0; a < N; ++a) {
        const int i = a + N * b;
        for (int a2 = 0; a2 < N; ++a2) {  // eta1 line
          const int j = a2 + N * b, ix = a * N + a2;
          s_at(0, i, j) += t.w[b] * t.skQ1[ix];
          s_at(1, i, j) += t.w[b] * t.skA1[ix];
        }
        for (int b2 = 0; b2 < N; ++b2) {  // eta2 line
          const int j = a + N * b2;
          s_at(1, i, j) += t.w[a] * t.skA2[b * N + b2];
        }
        rb_at(0, a, i) = t.lL[b] * t.Bf[0 * Nqf + a];
        rb_at(1, b, i) = t.lR[a] * t.Bf[1 * Nqf + b];
        rb_at(2, b, i) = t.lL[a] * t.Bf[2 * Nqf + b];
      }
  } else {
    for (int c = 0; c < N; ++c)
      for (int b = 0; b < N; ++b)
        for (int a = 0; a < N; ++a) {
          const int i = a + N * b + N * N * c;
          const double c0 = 0.5 * t.w[b] * t.w3[c], c1 = 0.5 * t.w[a] * t.w3[c],
                       c2 = 0.125 * t.w[a] * t.w[b] * (1.0 - t.eta[b]);
          for (int a2 = 0; a2 < N; ++a2) {  // eta1 line: S^(0), S^(1), S^(2)
            const int j = a2 + N * b + N * N * c, ix = a * N + a2;
            s_at(0, i, j) += c0 * t.skQ1[ix];
            s_at(1, i, j) += c0 * t.skA1[ix];
            s_at(2, i, j) += c0 * t.skA1[ix];
          }
          for (int b2 = 0; b2 < N; ++b2) {  // eta2 line: S^(1), S^(2)
            const int j = a + N * b2 + N * N * c, ix = b * N + b2;
            s_at(1, i, j) += c1 * t.skA2[ix];
            s_at(2, i, j) += c1 * t.skA3[ix];
          }
          for (int c2i = 0; c2i < N; ++c2i) {  // eta3 line: S^(2)
            const int j = a + N * b + N * N * c2i;
            s_at(2, i, j) += c2 * t.skA4[c * N + c2i];
          }
          rb_at(0, a + N * c, i) = t.lL[b] * t.Bf[0 * Nqf + a + N * c];
          rb_at(1, b + N * c, i) = t.lR[a] * t.Bf[1 * Nqf + b + N * c];
          rb_at(2, b + N * c, i) = t.lL[a] * t.Bf[2 * Nqf + b + N * c];
          for (int j4 = 0; j4 < N; ++j4)
            rb_at(3, a + N * j4, i) = t.l3L[c] * t.lint4[j4 * N + b] * t.Bf[3 * Nqf + a + N * j4];
        }
  }
}

// barycentric coordinates [M][d+1] of the degree-N node family (0: lattice, 1: warp & blend), rounded
std::vector<double> node_family_bary(int d, int N, int family) {
  std::vector<LD> b;
  node_bary(d, N, family, b);
  return rnd(b);
}

}  // namespace esb
