/*
 * es.h -- C ABI of the B200-native (sm_100a) entropy-stable modal DSEM right-hand side.
 *
 * Method: Montoya & Zingg, arXiv 2312.07874 (PAPER.md, cited as P:<line> [label]).
 *   es_rhs evaluates d u~/dt = M~^{-1} V^T r (P:446 [eq:dudt_modal]) with r the entropy-stable
 *   flux-differencing residual of P:520 [eq:entropy_stable] including the facet correction of P:525
 *   [eq:facet_correction], for the compressible Euler equations with Ranocha's
 *   entropy-conservative two-point flux (energy term per DESIGN.md reading R3) in the volume
 *   and facet-correction terms and the EC or ES (EC + local Lax-Friedrichs with Davis wave speed,
 *   P:491) interface flux.  Volume fluxes are evaluated line by line in collapsed coordinates
 *   (P:572), one evaluation per node pair on each eta_k line.
 *
 * Conventions (all functions):
 *   - reals are IEEE FP64; arrays are C-contiguous;
 *   - modal arrays are the LOCAL block u[k_local][e][i]: element k_local in [0, n_local), conserved
 *     variable e in {rho, rho v_1..rho v_d, E} (N_c = d+2), PKD mode i in [0, N_p*) in the
 *     alpha1-major nested order (for a1 in 0..p: for a2 in 0..p-a1: [for a3 in 0..p-a1-a2]);
 *   - "device pointer" = CUDA global memory of the context's device (e.g. torch tensor data_ptr());
 *     "host pointer" = ordinary or pinned host memory;
 *   - the caller owns every buffer it passes; the library copies what it keeps and owns all of its
 *     device allocations (geometry, tables, traces, RK state);
 *   - every function returns es_status; no C++ exception crosses the ABI.  After ES_ERR_CUDA or
 *     ES_ERR_NCCL the context is poisoned: every later call returns the same code.  Output buffers
 *     are undefined after a failed call.  es_last_error() returns a context-owned message;
 *   - calls on one context are not thread safe; one context per process / GPU;
 *   - es_rhs / es_step are asynchronous on the context stream unless opt.check_admissibility.
 */
#ifndef ES_B200_H
#define ES_B200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ES_OK = 0,
  ES_ERR_CONFIG = 2,        /* unsupported (dim, p) or inconsistent options */
  ES_ERR_INADMISSIBLE = 3,  /* rho <= 0 or p <= 0 at a projected node */
  ES_ERR_VERIFY = 4,        /* mesh check failed: J~ <= 0, unmatched face */
  ES_ERR_ARG = -1,          /* null / out-of-range argument */
  ES_ERR_CUDA = -5,
  ES_ERR_NCCL = -6,
  ES_ERR_OOM = -7
} es_status;

typedef struct es_context es_context;

/* Periodic conforming simplicial mesh.  Copied during es_setup. */
typedef struct {
  int dim;                          /* 2 (triangles) or 3 (tetrahedra) */
  int64_t n_elements;               /* global element count N_e */
  const int64_t* elem_vertices;     /* host [N_e][dim+1] periodic global vertex ids in CANONICAL
                                       order: ascending id, first two swapped if the corner simplex
                                       is negatively oriented (R11) */
  const double* elem_vertex_coords; /* host [N_e][dim+1][dim] unwrapped corner coordinates */
  const double* period;             /* host [dim] periodic lengths (fully periodic meshes) */
} es_mesh;

/* Geometry map (P:327 [eq:poly_mapping]): called ONCE by es_setup with the affine images of the
 * degree-p mapping nodes (es_options.mapping_nodes: equispaced lattice or warp & blend) of the local
 * elements, x_in host [n][dim] -> x_out host [n][dim].  The returned positions define the
 * isoparametric mapping.  */
typedef void (*es_map_fn)(void* user, int64_t n, const double* x_in, double* x_out);

typedef struct {
  double gamma;                         /* ratio of specific heats (1.4) */
  int interface_flux;                   /* 0 = entropy conservative, 1 = entropy stable with local
                                           Lax-Friedrichs dissipation, 2 = entropy stable
                                           with scalar dissipation on the entropy-variable jump (P:497,
                                           DESIGN.md R27), 3 = entropy stable with matrix dissipation
                                           (R28); other values: ES_ERR_CONFIG */
  int rank, world;                      /* local elements [rank*N_e/world, (rank+1)*N_e/world) */
  const unsigned char* nccl_unique_id;  /* 128-byte ncclUniqueId (world > 1), broadcast by caller;
                                           NULL with world > 1: the caller moves the halo itself
                                           (es_rhs_stage1 / es_halo_buffer / es_rhs_stage2) */
  void* cuda_stream;                    /* cudaStream_t to launch on; NULL = a library stream */
  int device;                           /* CUDA device ordinal */
  int check_admissibility;              /* 1: es_rhs synchronises and returns ES_ERR_INADMISSIBLE */
  int volume_mode;                      /* 0: line-wise flux differencing (the default);
                                           1: ablation -- one flux per operator S^(l) with a
                                           nonzero on the line, the paper's Eq. num_fluxes
                                           iteration; same result up to rounding;
                                           2: ablation -- brute force over every node pair with
                                           the dense operators, zeros included (SURVEY 8(f) rank
                                           2; O(N_q^2) per element, small configurations only);
                                           other values: ES_ERR_CONFIG */
  int mapping_nodes;                    /* node family of the isoparametric map (degree p_g = p) and of
                                           the 3D curl-metric interpolant (degree q + 1), P:845:
                                           0: equispaced barycentric lattice (R10, the
                                           default); 1: warp & blend -- Gauss-Lobatto-Legendre points
                                           on the edges, Warburton's blend with alpha = 0 inside
                                           (R32); other values: ES_ERR_CONFIG */
  int metric_storage;                   /* volume metric terms G_lm read by the flux kernel (P:595:
                                           "geometric information at each volume and facet
                                           quadrature node"): 0: nodal values
                                           (the default); 1: modal -- PKD coefficients V^T W G_lm
                                           (N_p* instead of N_q doubles per entry, 4.4x fewer bytes at
                                           p = 8 in 3D), expanded to G = V g~ in the flux kernel's
                                           prologue; exact up to rounding, the metric terms being
                                           polynomials of degree <= p (R33).  Applies to
                                           volume_mode 0 (the ablation kernels read the nodal copy,
                                           which setup keeps); other values: ES_ERR_CONFIG */
} es_options;

/* Builds tables, geometry (exact metrics in 2D, conservative curl metrics in 3D, P:345-364;
 * Jacobian interpolant P:448-452), connectivity and the halo plan; uploads everything to the
 * device.  p in [1, 10] for dim 2 and [1, 8] for dim 3 (q = p).  */
es_status es_setup(es_context** ctx, const es_mesh* mesh, int p, es_map_fn map, void* map_user,
                   const es_options* opt);
void es_destroy(es_context* ctx);
const char* es_last_error(const es_context* ctx);

/* Sizes: N_p*, N_q, N_qf per facet, local element count and first global element. */
es_status es_sizes(const es_context* ctx, int* Np, int* Nq, int* Nqf, int64_t* n_local,
                   int64_t* first_element);

/* d u~/dt for the local block: u_modal, dudt_modal device pointers [n_local][N_c][N_p*].
 * Includes the face-trace halo exchange (NCCL) when world > 1. */
es_status es_rhs(es_context* ctx, const double* u_modal, double* dudt_modal);
/* Same, with HOST buffers: host->device copy, es_rhs, device->host copy, synchronised. */
es_status es_rhs_host(es_context* ctx, const double* u_modal_host, double* dudt_modal_host);

/* Two-stage RHS for callers that move the face-trace halo themselves (world > 1 without NCCL, e.g.
 * several ranks in one process).  Stage 1: entropy projection of u_modal
 * (device) and packing of the boundary traces; *send_buf receives the device send buffer: faces
 * ordered by destination rank, then by (element, face) id, N_c*N_qf doubles each (counts from
 * es_plan).  es_halo_buffer: device buffer where the caller places the received faces, ordered by
 * source rank, then by the sender's (element, face) id.  Stage 2 (after the halo is in place and
 * the caller has ordered it before the context stream): interface fluxes and the flux kernel ->
 * dudt_modal (device).  All asynchronous on the context stream. */
es_status es_rhs_stage1(es_context* ctx, const double* u_modal, double** send_buf);
es_status es_halo_buffer(es_context* ctx, double** recv_buf);
es_status es_rhs_stage2(es_context* ctx, double* dudt_modal);

/* Library-owned RK state: copy in/out (device pointers, [n_local][N_c][N_p*]). */
es_status es_set_state(es_context* ctx, const double* u_modal);
es_status es_get_state(es_context* ctx, double* u_modal);
/* nsteps classical RK4 steps of size dt on the library state (R17). */
es_status es_step(es_context* ctx, double dt, int nsteps);

/* End to end through host buffers (the e2e measurement path): copies u_host (HOST, [n_local][N_c][N_p*],
 * pinned for an asynchronous copy) into the library state, advances nsteps classical RK4 steps of
 * size dt (es_step) and copies the state back into u_host_out (HOST).  Synchronous. */
es_status es_step_host(es_context* ctx, const double* u_host, double* u_host_out, double dt, int nsteps);

/* One or more explicit Runge-Kutta steps with a caller-supplied Butcher tableau (s <= 16 stages; A[s][s]
 * strictly lower triangular, row-major, b[s]; HOST arrays): U <- U + dt sum_j b_j k_j with
 * k_j = f(U + dt sum_{l<j} a_jl k_l), on the library state.  Passing the coefficients of Dormand-Prince
 * 8 (Hairer-Norsett-Wanner I, II.5 -- the paper's integrator) from a published table gives the
 * paper's time integration at a fixed step.  Allocates s state-sized slope buffers on first use.
 * Asynchronous (synchronous with check_admissibility). */
es_status es_step_erk(es_context* ctx, double dt, int s, const double* A, const double* b, int nsteps);

/* CUDA graphs for es_step (default on): with world == 1 and no per-kernel timing the launches of one
 * RK4 step are captured once per dt into a CUDA graph and replayed.  on = 0 launches them eagerly
 * (the same kernels and arguments: results are bitwise identical). */
es_status es_set_graphs(es_context* ctx, int on);
/* One Dormand-Prince 5(4) step of size dt on the library state (Hairer-Norsett-Wanner I, II.5; the
 * paper integrates with DP8 of the same family).  *err = sqrt(mean_i (e_i / (atol + rtol
 * max(|y0_i|, |y5_i|)))^2) over all modal coefficients of all ranks, e = y5 - y4 the embedded
 * estimate.  *accepted = (*err <= 1): the state advances to the 5th-order solution y5; otherwise it is
 * unchanged (the caller retries with a smaller dt).  First-same-as-last: f(y5) is reused by the next
 * call unless es_set_state / es_step intervene.  Allocates 8 state-sized buffers on first use.
 * Synchronous (reads err); ES_ERR_ARG for dt <= 0, negative tolerances or NULL outputs. */
es_status es_step_dp54(es_context* ctx, double dt, double rtol, double atol, double* err, int* accepted);

/* Entropy production sum_k sum_e w^T r = d/dt sum_k 1^T W J~ s, global over ranks,
 * its absolute scale sum |w_i r_i| (computed modally as sum |w~_i (V^T r)_i|), and the global
 * conservation residuals sum_k 1^T r^(e), conservation[N_c].  u_modal: device pointer.
 * Synchronous; includes an ncclAllReduce when world > 1.  Any output pointer may be NULL. */
es_status es_entropy_production(es_context* ctx, const double* u_modal, double* rate,
                                double* abs_scale, double* conservation);

/* Two-point flux evaluations per element and RHS (integers, exact): volume evaluations (line-wise
 * pairs, or per-operator evaluations with volume_mode 1), facet-correction pairs, the Eq.
 * num_fluxes count, interface evaluations per element. */
es_status es_flux_counts(const es_context* ctx, int64_t* volume_pairs_per_el,
                         int64_t* facet_pairs_per_el, int64_t* eq56_per_el,
                         double* interface_per_el);

/* Flux evaluations COUNTED IN THE KERNELS (P:563-567 Eq. num_fluxes; BASELINE north_star "integer
 * counts must match exactly"): runs one RHS on u_modal (device) with the counting instantiation of
 * the flux kernel (same arithmetic, per-element counters) and writes counts[n_local][4] (HOST):
 *   [0] volume two-point flux evaluations with a nonzero operator coefficient (line-wise pairs, or
 *       per-operator evaluations with volume_mode 1),
 *   [1] facet-correction evaluations (nonzeros of R^T B),
 *   [2] every evaluation the kernel's lanes issued, masked jobs included (idle-lane diagnostic),
 *   [3] interface flux evaluations (one per facet node of the element; both sides of a face count).
 * Synchronous.  volume_mode 2 (brute force) is not instrumented: ES_ERR_CONFIG. */
es_status es_count_fluxes(es_context* ctx, const double* u_modal, int64_t* counts);

/* Loopback groups (one-GPU emulation of world > 1, tests): ctxs[r] (r = 0..n-1) are the n ranks of one
 * mesh, each created with world = n, rank = r and nccl_unique_id = NULL, on one device in this process.
 * These calls run the complete multi-rank path of es_rhs / es_step / es_entropy_production -- K1, pack
 * of the boundary traces, interior-element interface fluxes overlapping the exchange, the wait, the
 * boundary-element interface fluxes, flux kernel, K3 -- with the NCCL send/recv replaced by one
 * cudaMemcpyAsync per (receiver, sender) pair on the receiver's communication stream, ordered after
 * the sender's pack by an event, and the allreduce by a host sum over ranks.  u[r] / dudt[r]: device
 * pointers of rank r's local block.  es_group_step advances every rank's library state (es_set_state).
 * Asynchronous except es_group_entropy_production (synchronous). */
es_status es_group_rhs(es_context** ctxs, int n, const double* const* u, double* const* dudt);
es_status es_group_step(es_context** ctxs, int n, double dt, int nsteps);
es_status es_group_entropy_production(es_context** ctxs, int n, const double* const* u, double* rate,
                                      double* abs_scale, double* conservation);

/* Linear-advection workload: du/dt + div(a u) = 0 with constant velocity a on the
 * context's mesh and geometry, in the skew-symmetric weak form of P:431-436 [eq:rhs_skew] (form 0; energy
 * stable on curved meshes) or the conservative form P:425-426 [eq:rhs_cons] (form 1), with the central
 * (flux_mode 0) or upwind (1) numerical flux, and the weight-adjusted inverse mass matrix.  The
 * scalar state is u_modal[n_local][N_p*] (device).  Single rank (ES_ERR_CONFIG otherwise).
 *   es_adv_configure: velocity a[dim], flux and form; allocates the workload's buffers.
 *   es_adv_rhs: du~/dt; energy (HOST, may be NULL) receives (sum_k u^T r, sum_k |u_i r_i|), the rate
 *     d/dt of sum_k u~^T M~ u~ / 2 and its scale (synchronous when energy != NULL).
 *   es_adv_step: nsteps classical RK4 steps (R17) of u_modal in place (asynchronous). */
es_status es_adv_configure(es_context* ctx, const double* a, int flux_mode, int form);
es_status es_adv_rhs(es_context* ctx, const double* u_modal, double* dudt_modal, double* energy);
es_status es_adv_step(es_context* ctx, double* u_modal, double dt, int nsteps);

/* Physical coordinates of the volume quadrature nodes, device pointer [n_local][N_q][dim]. */
es_status es_node_coords(es_context* ctx, double* x_dev);
/* Reference L2 projection u~ = V^T W u (M = I): u_nodal device [n_local][N_q][N_c] ->
 * u_modal device [n_local][N_c][N_p*].  (Initial data; R18.) */
es_status es_project_nodal(es_context* ctx, const double* u_nodal, double* u_modal);

/* Evaluation at the volume quadrature nodes u = V u~: u_modal device [n_local][N_c][N_p*]
 * -> u_nodal device [n_local][N_q][N_c].  (Error norms, output.) */
es_status es_eval_nodal(es_context* ctx, const double* u_modal, double* u_nodal);
/* Evaluation at arbitrary reference points (error norms with a rule of the caller's choice, e.g. the
 * degree-35 collapsed Gauss rule behind the paper's L2 errors): xi_host[npts][dim] (HOST) on the
 * reference simplex (vertices of P:177 / P:257).  Writes (device) u_out[n_local][npts][N_c] =
 * sum_k u~_k psi_k(xi) (PKD basis), and when non-NULL x_out[n_local][npts][dim] = x^(kappa)(xi)
 * (the degree-p_g mapping) and jac_out[n_local][npts] = det(dx/dxi) of that mapping (the
 * exact Jacobian, not J~).  u_modal: device.  Synchronous. */
es_status es_eval_points(es_context* ctx, const double* u_modal, int npts, const double* xi_host,
                         double* u_out, double* x_out, double* jac_out);

/* Quadrature weights of the volume nodes in physical space, W J~: device [n_local][N_q];
 * sum_k sum_i wj f(x_i) integrates f over the local elements (exact for the L2 norm of P_p data). */
es_status es_node_weights(es_context* ctx, double* wj);

/* Geometry of one local element copied to HOST buffers (tests): G [N_q][dim][dim] (G_lm),
 * Jn [N_f][N_qf][dim] = G^T nhat at facet nodes, Jt [N_q] = J~.  NULL = skip. */
es_status es_element_geometry(es_context* ctx, int64_t local_element, double* G, double* Jn,
                              double* Jt);

/* Host-only (no GPU needed): the reference tables the kernels use for (dim, p), copied to the host
 * buffer out (capacity cap doubles); *n receives the length.  Names: "eta","w","eta3","w3" [n];
 * "skQ1","skA1","skA2","skA3","skA4" [n][n] skew line operators; "lL","lR","l3L" [n];
 * "lint4" [n][n]; "psi1" [n][n], "psi2","psi3" [n][n][n]; "Wvol" [N_q]; "Bf" [N_f][N_qf];
 * "xi_vol" [N_q][dim].  Returns ES_ERR_ARG for an unknown name or too small a buffer. */
es_status es_ref_table(int dim, int p, const char* name, double* out, int64_t cap, int64_t* n);

/* Host-only: connectivity and halo plan of rank `rank` of `world` (no GPU).  face_slot [n_local][N_f]
 * (trace slot of the neighbour face: local slots e*N_f+z, halo slots n_local*N_f + h),
 * face_reflect [n_local][N_f], send_slots [n_send], send_count/recv_count [world]; any output may be
 * NULL; *n_send, *n_halo receive the sizes. */
es_status es_plan(int dim, int64_t n_elements, const int64_t* elem_vertices, int rank, int world,
                  int64_t* face_slot, int* face_reflect, int64_t* send_slots, int64_t* send_count,
                  int64_t* recv_count, int64_t* n_send, int64_t* n_halo);

/* Synchronise the context stream (and report asynchronous CUDA errors). */
es_status es_synchronize(es_context* ctx);
/* Stream the context launches on (cudaStream_t as void*). */
void* es_stream(const es_context* ctx);

/* Kernel launch accounting: number of library kernels launched since the last reset. */
int64_t es_launch_count(const es_context* ctx);
void es_reset_launch_count(es_context* ctx);

/* Per-launch timing of the kernels (CUDA events on the context stream): es_timing_enable(ctx, 1)
 * starts recording; es_timing_read returns the summed milliseconds and the number of launches of
 * each kernel class since enabling: 0 = entropy projection / trace kernel, 1 = flux-differencing
 * + lifting + inverse-mass kernel, 2 = interface-flux kernel. */
es_status es_timing_enable(es_context* ctx, int on);
es_status es_timing_read(es_context* ctx, int kernel_class, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif
