/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the entropy-stable modal DSEM right-hand side of
 * Montoya & Zingg, "Efficient entropy-stable discontinuous spectral-element methods using
 * tensor-product summation-by-parts operators on triangles and tetrahedra" (arXiv 2312.07874).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load
 * this library.  It shares no code, header, table or helper with the CUDA product path in
 * paper_2312_07874_b200/ and neither includes the other.
 *
 * Citation format: P:<line> = /root/reference/PAPER.md line, followed by the equation label.
 * Readings of the paper where it is silent/garbled are numbered as in DESIGN.md section 3 (R1..R33).
 *
 * All reals are IEEE FP64, compiled with -O2 -ffp-contract=off (no FMA contraction).
 * Layout of modal arrays (same as the product ABI, include/es.h): u[element][variable e][mode k],
 * with the PKD multi-index order pi = alpha1-major nested (R9).
 * Volume node order sigma: eta1 fastest, then eta2, then eta3 (R9).  Facet node order sigma_f:
 * eta_f1 fastest (R9).
 */
#ifndef ES_ORACLE_H
#define ES_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- 1D building blocks, P:139-164 ---- */
double ora_jacobi(int n, double a, double b, double x);          /* normalised P_n^(a,b) */
double ora_jacobi_deriv(int n, double a, double b, double x);
int ora_gauss_jacobi(int q, double a, double b, double* x, double* w); /* q+1 Gauss nodes */
void ora_lagrange_diff(int n, const double* nodes, double* D);  /* D[i*n+j] = l_j'(x_i) */

/* ---- reference operators, P:166-300 (dense) ----
 * ora_ref_sizes -> out[0..4] = n=q+1, Nq, Nf, Nqf, Np.
 * ora_ref_get(name): "eta1","w1","eta3","w3" [n]; "xi" [Nq][d]; "W" [Nq]; "xif" [Nf][Nqf][d];
 *   "B" [Nf][Nqf]; "nhat" [Nf][d]; "D","Q","E","S" [d][Nq][Nq]; "R" [Nf][Nqf][Nq]; "V" [Nq][Np];
 *   "alpha" [Np][d] (as doubles).  Returns 0 on success, -1 on unknown name. */
void ora_ref_sizes(int d, int q, int p, int* out);
int ora_ref_get(int d, int q, int p, const char* name, double* out);
/* PKD basis and gradient at arbitrary points of the reference simplex (Cartesian
 * homogenised form, valid at the collapsed vertex too).  vals[npts][Np], grads[npts][Np][d]. */
void ora_pkd_eval(int d, int p, int npts, const double* xi, double* vals, double* grads);

/* ---- physics, P:805-841 and SURVEY App. B (R3, R5, R7) ----
 * States are conservative U[n][d+2].  */
void ora_entropy_vars(int d, double gamma, int n, const double* U, double* W);
void ora_cons_from_entropy(int d, double gamma, int n, const double* W, double* U);
void ora_euler_flux(int d, double gamma, int n, const double* U, const double* nvec, double* F);
void ora_ec_flux(int d, double gamma, int n, const double* Ua, const double* Ub, const double* nvec,
                 double* F);
void ora_es_flux(int d, double gamma, int n, const double* Ua, const double* Ub, const double* nunit,
                 double* F);
double ora_wave_speed(int d, double gamma, const double* Ua, const double* Ub, const double* nunit);
/* du/dw [n][d+2][d+2] (R27) and the entropy-jump dissipative interface flux (R27) */
void ora_dudw(int d, double gamma, int n, const double* U, double* A);
void ora_ej_flux(int d, double gamma, int n, const double* Ua, const double* Ub, const double* nunit,
                 double* F);
/* matrix-dissipation interface flux (R28) */
void ora_md_flux(int d, double gamma, int n, const double* Ua, const double* Ub, const double* nunit,
                 double* F);
double ora_ln_mean(double x, double y);
double ora_inv_ln_mean(double x, double y);
void ora_entropy(int d, double gamma, int n, const double* U, double* S, double* Fent /*[n][d]*/);

/* ---- mesh, geometry and RHS, P:322-364, P:439-534, P:538-595 ---- */
typedef void (*ora_map_fn)(void* user, int64_t n, const double* x_in, double* x_out);
typedef struct ora_mesh ora_mesh;
typedef struct {
  int64_t volume_pairs;      /* two-point flux evaluations in the volume term */
  int64_t facet_pairs;       /* two-point flux evaluations in the facet correction */
  int64_t interface_evals;   /* numerical interface flux evaluations (per element side) */
  int64_t series_branch;     /* log-mean evaluations taking the Taylor-series branch (R5) */
  int64_t log_branch;        /* log-mean evaluations taking the log branch */
  int64_t n_elements;        /* elements whose RHS was evaluated */
  double entropy_rate;       /* sum_k sum_e w^T r over evaluated elements */
  double entropy_abs;        /* sum_k sum_e sum_i |w_i r_i| */
  double conservation[5];    /* sum_k sum_i r_i^(e) */
  int inadmissible;          /* 1 if rho<=0 or p<=0 met at any projected node */
} ora_stats;

/* Creates the mesh: elem_vertices [ne][d+1] global ids in canonical order (R11),
 * elem_vertex_coords [ne][d+1][d] unwrapped corner coordinates, period [d].  map is called once with
 * all affine mapping-node images of the ACTIVE elements (n points).  active = NULL -> all elements;
 * otherwise geometry is built only for the listed elements and their face neighbours.
 * Returns NULL and prints the reason on failure (J<=0, unmatched face, bad permutation). */
ora_mesh* ora_mesh_create(int d, int p, int64_t ne, const int64_t* elem_vertices,
                          const double* elem_vertex_coords, const double* period, ora_map_fn map,
                          void* user, double gamma, int64_t n_active, const int64_t* active);
/* as ora_mesh_create with the mapping / curl-interpolation node family: 0 = equispaced lattice
 * (R10), 1 = warp & blend (R32) */
ora_mesh* ora_mesh_create2(int d, int p, int64_t ne, const int64_t* elem_vertices,
                           const double* elem_vertex_coords, const double* period, ora_map_fn map,
                           void* user, double gamma, int64_t n_active, const int64_t* active, int node_family);
/* node set of degree N (family as above): xi [M][d], lam [M][d+1] (either may be NULL); returns M */
int ora_nodes(int d, int N, int family, double* xi, double* lam);
void ora_mesh_destroy(ora_mesh* m);
/* geometric factors of one element: G [Nq][d][d] (G_lm), Gf [Nf][Nqf][d][d], Jt [Nq], Jn
 * [Nf][Nqf][d], xq [Nq][d]; any pointer may be NULL. Returns 0, or -1 if geometry not built. */
int ora_mesh_geometry(const ora_mesh* m, int64_t elem, double* G, double* Gf, double* Jt,
                      double* Jn, double* xq);
/* modal (compressed) metric storage, SURVEY 8(f) rank 4 / P:595: gm [d*d][Np] = V^T W G_lm of one
 * element (row l*d + m; exact L2 projection, the metric terms being polynomials of degree <= p).
 * Returns 0, or -1 if geometry not built. */
int ora_metric_modal(const ora_mesh* m, int64_t elem, double* gm);
/* replaces the volume metric G of every element by V (V^T W G), i.e. the values a modal store
 * reproduces at the volume nodes (facet metrics unchanged); afterwards ora_rhs runs on them. */
int ora_mesh_use_modal_metrics(ora_mesh* m);
/* connectivity: nbr[ne][Nf], nbr_face[ne][Nf], reflect[ne][Nf] */
void ora_mesh_conn(const ora_mesh* m, int64_t* nbr, int* nbr_face, int* reflect);
/* modal L2 projection u_modal = V^T W u_nodal (R18) for the listed elements.
 * u_nodal [ne][Nq][Nc] (only listed rows read), u_modal [ne][Nc][Np] (only listed rows written). */
void ora_project(const ora_mesh* m, int64_t n_el, const int64_t* elems, const double* u_nodal,
                 double* u_modal);
/* RHS: dudt [ne][Nc][Np] for the listed elements (NULL list = all).  flux_mode 0 = EC, 1 = ES
 * (EC + LLF/Davis), 2 = EC + entropy-jump scalar dissipation (R27), 3 = EC + matrix
 * dissipation (R28).  variant 0 = Eq. num_fluxes nonzero loops, 1 = line-wise pairing
 * (P:572), 2 = dense brute force (all i,j), 3 = hybridised SBP (Chan-Wilcox eq. 35).
 * nthreads <= 0 -> OpenMP default.  Returns 0, or 3 if an inadmissible state was met. */
int ora_rhs(const ora_mesh* m, const double* u_modal, double* dudt, int flux_mode, int variant,
            int64_t n_out, const int64_t* out_elems, int nthreads, ora_stats* stats);
/* nsteps classical RK4 steps of size dt on all elements (R17), in place. */
int ora_rk4(const ora_mesh* m, double* u_modal, double dt, int nsteps, int flux_mode, int nthreads);
/* Dormand-Prince 5(4) (Hairer-Norsett-Wanner I, II.5): tableau (c[7], a[7][7], b[7], bh[7]) and one step
 * of size dt from u_modal (unchanged) -> u5 (5th order) and the scaled RMS error estimate *err */
void ora_dp54_tableau(double* c, double* a, double* b, double* bh);
int ora_dp54(const ora_mesh* m, const double* u_modal, double dt, double rtol, double atol, int flux_mode,
             int nthreads, double* u5, double* err);

/* Linear advection du/dt + div(a u) = 0: scalar modal state
 * u_modal[ne][Np], constant velocity a[dim]; form 0 = skew-symmetric [eq:rhs_skew], 1 = conservative
 * [eq:rhs_cons]; flux_mode 0 central, 1 upwind.  dudt[ne][Np] = M~^{-1} V^T r; energy[2] = (sum u^T r,
 * sum |u_i r_i|).  Requires geometry for every element. */
int ora_advection_rhs(const ora_mesh* m, const double* u_modal, const double* a, int flux_mode, int form,
                      double* dudt, double* energy);

#ifdef __cplusplus
}
#endif
#endif
