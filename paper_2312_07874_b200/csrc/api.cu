// api.cpp -- the C ABI declared in include/es.h: context, setup, RHS / RK4 / entropy drivers,
// NCCL face-trace halo exchange.  Product code (no CPU fallback: every step runs in the kernels).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "es.h"
#include "geometry.cuh"
#include "internal.h"
#include "kernels.cuh"
#include "xform3.cuh"
#include "advect.cuh"

namespace esb {
cudaError_t launch_project_2d(int n, const DevRef& R, const ProjArgs& A, cudaStream_t st);
cudaError_t launch_project_3d(int n, const DevRef& R, const ProjArgs& A, cudaStream_t st);
cudaError_t launch_rhs_2d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st);
cudaError_t launch_rhs_3d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st);
cudaError_t launch_projnodal_2d(int n, const DevRef& R, int64_t ne, const double* un, double* um, cudaStream_t st);
cudaError_t launch_projnodal_3d(int n, const DevRef& R, int64_t ne, const double* un, double* um, cudaStream_t st);
cudaError_t launch_evalnodal_2d(int n, const DevRef& R, int64_t ne, const double* um, double* un, cudaStream_t st);
cudaError_t launch_evalnodal_3d(int n, const DevRef& R, int64_t ne, const double* um, double* un, cudaStream_t st);
cudaError_t upload_psi_3d(int n, const double* p1, const double* p2, const double* p3);
cudaError_t launch_rhs_count_2d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st);
cudaError_t launch_rhs_count_3d(int n, const DevRef& R, const RhsArgs& A, cudaStream_t st);
cudaError_t launch_wadj_3d(int n, const WadjArgs& A, cudaStream_t st);
cudaError_t upload_psi_3d_k1(int n, const double* p1, const double* p2, const double* p3);
cudaError_t upload_psi_adv_3d(int n, const double* p1, const double* p2, const double* p3);
cudaError_t launch_adv_2d(int n, const DevRef& R, const AdvArgs& A, cudaStream_t st);
cudaError_t launch_adv_3d(int n, const DevRef& R, const AdvArgs& A, cudaStream_t st);
cudaError_t launch_wjinv_permute_3d(int n, const double* geo_vol, int gvs, int row, int64_t ne, double* out,
                                    cudaStream_t st);
}  // namespace esb

using namespace esb;

struct TimedEvent {
  cudaEvent_t a, b;
  int cls;
};

struct es_context {
  std::string err;
  es_status poisoned = ES_OK;
  int d = 0, p = 0, n = 0, Nq = 0, Nqf = 0, Nf = 0, Np = 0, NC = 0;
  int64_t ne = 0, first = 0, nloc = 0, nslots = 0;
  double gamma = 1.4, c0 = 0.0;
  int es = 1, check_adm = 0, rank = 0, world = 1, device = 0;
  cudaStream_t stream = nullptr, comm_stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev_packed = nullptr, ev_comm = nullptr;
  RefTables T;
  MeshPlan plan;
  DevRef R{};
  void* d_tables = nullptr;
  double *geo_vol = nullptr, *geo_face = nullptr, *xq = nullptr, *jt = nullptr;
  double *prim = nullptr, *trace = nullptr, *wt = nullptr, *part = nullptr, *red = nullptr;
  double *rbuf = nullptr, *wjk3 = nullptr;  // 3D: nodal residual for K3, W / J~ in K3's layout
  double* xmapv = nullptr;                   // [nloc][Npg][dim] mapping-node positions (es_eval_points)
  unsigned long long* dcounts = nullptr;    // es_count_fluxes: per-element flux-evaluation counters
  bool counting = false;
  // CUDA graph of one classical RK4 step (4 right-hand sides, 12-16 launches) replayed by es_step
  cudaGraphExec_t step_graph = nullptr;
  double step_graph_dt = 0.0;
  int64_t step_graph_launches = 0;
  bool use_graphs = true;
  // es_step_erk: slopes of a caller-supplied explicit Runge-Kutta tableau, and the next-state buffer
  std::vector<double*> erk_k;
  double* erk_y = nullptr;
  // linear-advection workload (es_adv_*): velocity, flux, form, buffers
  double adv_a[3] = {0, 0, 0};
  int adv_flux = 1, adv_form = 0;
  bool adv_ready = false;
  double *adv_unod = nullptr, *adv_trace = nullptr, *adv_X = nullptr, *adv_acc = nullptr, *adv_us = nullptr,
         *adv_part = nullptr;
  int num_sms = 148, proj_ctas = 296;
  bool external = false;
  int eq56 = 0;   // volume_mode 1: per-operator fluxes (Eq. num_fluxes ablation)
  int dense = 0;  // volume_mode 2: brute force over all node pairs (dense operators)
  int metric_modal = 0;    // es_options.metric_storage 1: volume metric as PKD coefficients
  double* gmod = nullptr;  // [nloc][even(NG Np)] PKD coefficients of G_lm (metric_modal)
  double *sdense = nullptr, *rbdense = nullptr;
  int64_t *face_slot = nullptr, *d_interior = nullptr, *d_boundary = nullptr, *d_send = nullptr;
  int* face_reflect = nullptr;
  int* bad = nullptr;
  double *U = nullptr, *ACC = nullptr, *US = nullptr, *hin = nullptr, *hout = nullptr, *send_buf = nullptr;
  double* dpk[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // DP5(4) stage slopes
  double *dpy = nullptr, *dppart = nullptr;  // DP5(4) 5th-order solution, error partials
  bool dp_fsal = false;                      // dpk[0] holds f(U) (first same as last)
  ncclComm_t comm = nullptr;
  int64_t launches = 0;
  bool timing = false;
  long long* dbg = nullptr;  // ES_PHASE_TIMING diagnostics
  std::vector<double> psig_doubles;  // host copy of the padded psi tables (DevRef::psig)
  std::vector<TimedEvent> tev;
  std::vector<cudaEvent_t> ev_pool;
  std::vector<cudaEvent_t> pipe_ev;  // es_step_host pipeline: per chunk, copy done / kernel done
  std::vector<int> pipe_dep;         // per chunk: the last chunk holding a face neighbour of its elements
  int64_t* d_iota = nullptr;         // 0 .. nloc-1 (element lists of the pipeline's chunks)
};

namespace {

es_status fail(es_context* c, es_status s, const std::string& m) {
  if (c) {
    c->err = m;
    if (s == ES_ERR_CUDA || s == ES_ERR_NCCL) c->poisoned = s;
  }
  return s;
}
#define CK(x)                                                                                     \
  do {                                                                                            \
    cudaError_t _e = (x);                                                                         \
    if (_e != cudaSuccess)                                                                        \
      return fail(c, _e == cudaErrorMemoryAllocation ? ES_ERR_OOM : ES_ERR_CUDA,                  \
                  std::string(#x) + ": " + cudaGetErrorString(_e));                               \
  } while (0)
#define NK(x)                                                                                     \
  do {                                                                                            \
    ncclResult_t _r = (x);                                                                        \
    if (_r != ncclSuccess) return fail(c, ES_ERR_NCCL, std::string(#x) + ": " + ncclGetErrorString(_r)); \
  } while (0)
#define POISON_CHECK()                            \
  do {                                            \
    if (!c) return ES_ERR_ARG;                    \
    if (c->poisoned != ES_OK) return c->poisoned; \
  } while (0)

cudaEvent_t get_event(es_context* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

template <class T>
cudaError_t upload(T** dst, const std::vector<T>& v) {
  if (v.empty()) {
    *dst = nullptr;
    return cudaSuccess;
  }
  cudaError_t e = cudaMalloc((void**)dst, v.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
}

// pack the reference tables into one device allocation
es_status upload_tables(es_context* c) {
  const RefTables& t = c->T;
  std::vector<char> blob;
  std::vector<std::pair<size_t, int>> offs;  // (offset, kind)
  auto add_d = [&](const std::vector<double>& v) {
    size_t off = (blob.size() + 255) / 256 * 256;
    blob.resize(off + std::max<size_t>(v.size(), 1) * sizeof(double), 0);
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(double));
    return off;
  };
  auto add_i = [&](const std::vector<int>& v) {
    size_t off = (blob.size() + 255) / 256 * 256;
    blob.resize(off + std::max<size_t>(v.size(), 1) * sizeof(int), 0);
    if (!v.empty()) std::memcpy(blob.data() + off, v.data(), v.size() * sizeof(int));
    return off;
  };
  std::vector<int> mode_pr(t.Np), mode_last(t.Np);
  for (size_t pr = 0; pr < t.pair_off.size(); ++pr) {
    int cnt = (pr + 1 < t.pair_off.size() ? t.pair_off[pr + 1] : t.Np) - t.pair_off[pr];
    for (int k = 0; k < cnt; ++k) {
      mode_pr[t.pair_off[pr] + k] = (int)pr;
      mode_last[t.pair_off[pr] + k] = k;
    }
  }
  size_t o_eta = add_d(t.eta), o_w = add_d(t.w), o_eta3 = add_d(t.eta3), o_w3 = add_d(t.w3);
  size_t o_q1 = add_d(t.skQ1), o_a1 = add_d(t.skA1), o_a2 = add_d(t.skA2), o_a3 = add_d(t.skA3), o_a4 = add_d(t.skA4);
  size_t o_lL = add_d(t.lL), o_lR = add_d(t.lR), o_l3 = add_d(t.l3L), o_li4 = add_d(t.lint4);
  size_t o_p1 = add_d(t.psi1), o_p2 = add_d(t.psi2), o_p3 = add_d(t.psi3);
  size_t o_pa1 = add_i(t.pair_a1), o_pa2 = add_i(t.pair_a2), o_poff = add_i(t.pair_off), o_mpr = add_i(mode_pr),
         o_ml = add_i(mode_last);
  size_t o_B = add_d(t.Bf), o_nh = add_d(t.nhat), o_W = add_d(t.Wvol);
  // the psi tables in the padded layout of stage_psi / psi_tables (kernels.cuh) for kernels that read
  // them from global memory (L1) instead of staging them in shared memory (the slim K1)
  {
    const int n = t.n, NP = (n + 1) & ~1, npair = (int)t.pair_a1.size();
    const int nd = n * NP + n * n * NP + (t.d == 3 ? n * n * NP : 0) + 48;  // + PSPAD
    std::vector<double> pg(nd + (3 * npair + 1) / 2 + 1, 0.0);
    for (int r = 0; r < n; ++r)
      for (int q = 0; q < n; ++q) pg[(size_t)r * NP + q] = t.psi1[(size_t)r * n + q];
    for (int r = 0; r < n * n; ++r)
      for (int q = 0; q < n; ++q) {
        pg[(size_t)n * NP + (size_t)r * NP + q] = t.psi2[(size_t)r * n + q];
        if (t.d == 3) pg[(size_t)(n + n * n) * NP + (size_t)r * NP + q] = t.psi3[(size_t)r * n + q];
      }
    int* pi = reinterpret_cast<int*>(pg.data() + nd);
    for (int k = 0; k < npair; ++k) {
      pi[k] = t.pair_a1[k];
      pi[npair + k] = t.pair_a2[k];
      pi[2 * npair + k] = t.pair_off[k];
    }
    c->psig_doubles = pg;
  }
  size_t o_pg = add_d(c->psig_doubles);
  char* d = nullptr;
  CK(cudaMalloc((void**)&d, blob.size()));
  CK(cudaMemcpy(d, blob.data(), blob.size(), cudaMemcpyHostToDevice));
  c->d_tables = d;
  auto P = [&](size_t o) { return (const double*)(d + o); };
  auto I = [&](size_t o) { return (const int*)(d + o); };
  c->R = DevRef{P(o_eta), P(o_w), P(o_eta3), P(o_w3), P(o_q1), P(o_a1), P(o_a2), P(o_a3), P(o_a4),
                P(o_lL), P(o_lR), P(o_l3), P(o_li4), P(o_p1), P(o_p2), P(o_p3),
                I(o_pa1), I(o_pa2), I(o_poff), I(o_mpr), I(o_ml), P(o_B), P(o_nh), P(o_W), P(o_pg)};
  return ES_OK;
}

cudaError_t run_project(es_context* c, const double* u, int64_t n, const int64_t* list, double* wt) {
  ProjArgs A{n, list, u, c->geo_vol, c->prim, c->trace, wt, c->bad, c->gamma, c->dbg ? c->dbg + 4096 * 16 : nullptr,
             c->proj_ctas};
  c->launches++;
  return c->d == 2 ? launch_project_2d(c->n, c->R, A, c->stream) : launch_project_3d(c->n, c->R, A, c->stream);
}

// K2 (interface fluxes, line-wise flux differencing, facet correction, lifting; + the 2D epilogue) on
// n elements (all, or an element list)
cudaError_t run_k2(es_context* c, RhsArgs A, int64_t n, const int64_t* list) {
  A.n_elem = n;
  A.elem_list = list;
  if (n <= 0) return cudaSuccess;
  TimedEvent te{};
  if (c->timing) {
    te = {get_event(c), get_event(c), 1};
    cudaEventRecord(te.a, c->stream);
  }
  c->launches++;
  if (c->counting) A.counts = c->dcounts;
  cudaError_t e = c->counting ? (c->d == 2 ? launch_rhs_count_2d(c->n, c->R, A, c->stream)
                                           : launch_rhs_count_3d(c->n, c->R, A, c->stream))
                              : (c->d == 2 ? launch_rhs_2d(c->n, c->R, A, c->stream)
                                           : launch_rhs_3d(c->n, c->R, A, c->stream));
  if (c->timing) {
    cudaEventRecord(te.b, c->stream);
    c->tev.push_back(te);
  }
  return e;
}

// 3D: weight-adjusted inverse and the RK / entropy epilogue, batched over all local elements (K3)
cudaError_t run_k3(es_context* c, const RhsArgs& A) {
  if (c->d == 2) return cudaSuccess;
  WadjArgs W{c->nloc, c->rbuf, c->wjk3, A.mode, A.out, A.u0, A.acc, A.ustage, A.dt, A.wt, A.part, A.c0};
  TimedEvent t3{};
  if (c->timing) {
    t3 = {get_event(c), get_event(c), 3};
    cudaEventRecord(t3.a, c->stream);
  }
  c->launches++;
  cudaError_t e = launch_wadj_3d(c->n, W, c->stream);
  if (c->timing) {
    cudaEventRecord(t3.b, c->stream);
    c->tev.push_back(t3);
  }
  return e;
}

RhsArgs base_rhs_args(es_context* c) {
  RhsArgs A{};
  A.prim = c->prim;
  A.trace = c->trace;
  A.geo_vol = c->geo_vol;
  A.geo_face = c->geo_face;
  A.face_slot = c->face_slot;
  A.face_reflect = c->face_reflect;
  A.gamma = c->gamma;
  A.es = c->es;
  A.c0 = c->c0;
  A.dbg = c->dbg;
  A.max_ctas = c->num_sms;
  A.eq56 = c->eq56;
  A.sdense = c->sdense;
  A.rbdense = c->rbdense;
  A.nhat = c->R.nhat;
  A.rbuf = c->rbuf;
  A.gmod = c->gmod;
  return A;
}

// first half of a right-hand side: entropy projection and, with remote neighbours, the packed
// boundary traces (send buffer ordered by destination rank)
es_status rhs_first(es_context* c, const double* u, double* wt) {
  TimedEvent te{};
  if (c->timing) {
    te = {get_event(c), get_event(c), 0};
    cudaEventRecord(te.a, c->stream);
  }
  CK(run_project(c, u, c->nloc, nullptr, wt));
  if (c->timing) {
    cudaEventRecord(te.b, c->stream);
    c->tev.push_back(te);
  }
  if (c->world > 1) {
    const int per_face = c->NC * c->Nqf;
    const int64_t nsend = (int64_t)c->plan.send_slots.size();
    CK(launch_pack(c->trace, c->d_send, nsend, per_face, c->send_buf, c->stream));
    c->launches++;
  }
  return ES_OK;
}

// second half: interface fluxes (halo slots filled) and the flux-differencing kernel
es_status rhs_second(es_context* c, RhsArgs A) {
  CK(run_k2(c, A, c->nloc, nullptr));
  CK(run_k3(c, A));
  return ES_OK;
}

// One right-hand side in three phases; with world > 1:
//   (a) projection K1 on all local elements, pack of the boundary traces, the communication stream
//       waits for the pack;
//   (b) the halo exchange on the communication stream: NCCL grouped send/recv (rhs_phase_b_nccl), or
//       for a group of contexts in one process on one device one cudaMemcpyAsync per (receiver,
//       sender) pair (rhs_phase_b_loopback, es_group_*);
//   (c) interface fluxes of elements without remote neighbours (overlapping the exchange), wait for
//       the exchange, interface fluxes of the boundary elements, flux kernel (+ K3 in 3D).
// With world > 1 the projection runs on the boundary elements (those with a remote neighbour) first,
// so that their traces are packed and the exchange starts while K1 runs on the interior elements.
es_status rhs_phase_a(es_context* c, const double* u, double* wt) {
  if (c->world == 1) return rhs_first(c, u, wt);
  TimedEvent te{};
  if (c->timing) {
    te = {get_event(c), get_event(c), 0};
    cudaEventRecord(te.a, c->stream);
  }
  CK(run_project(c, u, (int64_t)c->plan.boundary.size(), c->d_boundary, wt));
  const int per_face = c->NC * c->Nqf;
  const int64_t nsend = (int64_t)c->plan.send_slots.size();
  CK(launch_pack(c->trace, c->d_send, nsend, per_face, c->send_buf, c->stream));
  c->launches++;
  CK(cudaEventRecord(c->ev_packed, c->stream));
  CK(cudaStreamWaitEvent(c->comm_stream, c->ev_packed, 0));
  CK(run_project(c, u, (int64_t)c->plan.interior.size(), c->d_interior, wt));
  if (c->timing) {
    cudaEventRecord(te.b, c->stream);
    c->tev.push_back(te);
  }
  return ES_OK;
}

es_status rhs_phase_b_nccl(es_context* c) {
  const int per_face = c->NC * c->Nqf;
  NK(ncclGroupStart());
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank) continue;
    if (c->plan.send_count[r] > 0)
      NK(ncclSend(c->send_buf + c->plan.send_offset[r] * per_face, (size_t)(c->plan.send_count[r] * per_face),
                  ncclDouble, r, c->comm, c->comm_stream));
    if (c->plan.recv_count[r] > 0)
      NK(ncclRecv(c->trace + (c->nloc * c->Nf + c->plan.recv_offset[r]) * per_face,
                  (size_t)(c->plan.recv_count[r] * per_face), ncclDouble, r, c->comm, c->comm_stream));
  }
  NK(ncclGroupEnd());
  CK(cudaEventRecord(c->ev_comm, c->comm_stream));
  return ES_OK;
}

// loopback transport: the receiver copies each sender's packed block (after the sender's pack)
es_status rhs_phase_b_loopback(es_context* c, es_context* const* group) {
  const int per_face = c->NC * c->Nqf;
  for (int r = 0; r < c->world; ++r) {
    if (r == c->rank || c->plan.recv_count[r] == 0) continue;
    es_context* s = group[r];
    CK(cudaStreamWaitEvent(c->comm_stream, s->ev_packed, 0));
    CK(cudaMemcpyAsync(c->trace + (c->nloc * c->Nf + c->plan.recv_offset[r]) * per_face,
                       s->send_buf + s->plan.send_offset[c->rank] * per_face,
                       (size_t)c->plan.recv_count[r] * per_face * sizeof(double), cudaMemcpyDeviceToDevice,
                       c->comm_stream));
  }
  CK(cudaEventRecord(c->ev_comm, c->comm_stream));
  return ES_OK;
}

es_status rhs_phase_c(es_context* c, RhsArgs A) {
  if (c->world == 1) return rhs_second(c, A);
  // the flux kernel on elements without remote neighbours overlaps the exchange (SURVEY 8(e),
  // north_star: "overlapped with the volume kernel"), then the boundary elements, then K3 on all
  CK(run_k2(c, A, (int64_t)c->plan.interior.size(), c->d_interior));
  CK(cudaStreamWaitEvent(c->stream, c->ev_comm, 0));
  CK(run_k2(c, A, (int64_t)c->plan.boundary.size(), c->d_boundary));
  CK(run_k3(c, A));
  return ES_OK;
}

// one right-hand side of one context (NCCL transport when world > 1)
es_status rhs_pass(es_context* c, const double* u, RhsArgs A, double* wt) {
  if (c->external) return fail(c, ES_ERR_CONFIG, "world > 1 without NCCL: use es_rhs_stage1 / es_rhs_stage2 or es_group_*");
  es_status s = rhs_phase_a(c, u, wt);
  if (s != ES_OK) return s;
  if (c->world > 1 && (s = rhs_phase_b_nccl(c)) != ES_OK) return s;
  return rhs_phase_c(c, A);
}

es_status check_bad(es_context* c) {
  int h = 0;
  CK(cudaMemcpyAsync(&h, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (h) {
    CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
    return fail(c, ES_ERR_INADMISSIBLE, "inadmissible state (rho <= 0 or p <= 0) at a projected node");
  }
  return ES_OK;
}

}  // namespace

extern "C" {

const char* es_last_error(const es_context* c) { return c ? c->err.c_str() : "null context"; }

void es_destroy(es_context* c) {
  if (!c) return;
  if (c->device >= 0) cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (void* p : {(void*)c->d_tables, (void*)c->geo_vol, (void*)c->geo_face, (void*)c->xq, (void*)c->jt,
                  (void*)c->prim, (void*)c->trace, (void*)c->wt, (void*)c->part, (void*)c->red,
                  (void*)c->face_slot, (void*)c->d_interior, (void*)c->d_boundary, (void*)c->d_send, (void*)c->d_iota,
                  (void*)c->face_reflect, (void*)c->bad, (void*)c->U, (void*)c->ACC, (void*)c->US,
                  (void*)c->hin, (void*)c->hout, (void*)c->send_buf, (void*)c->dbg,
                  (void*)c->dpy, (void*)c->dppart, (void*)c->sdense, (void*)c->rbdense, (void*)c->rbuf,
                  (void*)c->wjk3, (void*)c->dcounts, (void*)c->xmapv, (void*)c->adv_unod, (void*)c->adv_trace,
                  (void*)c->adv_X, (void*)c->adv_acc, (void*)c->adv_us, (void*)c->adv_part, (void*)c->gmod})
    if (p) cudaFree(p);
  for (double* p : c->dpk)
    if (p) cudaFree(p);
  for (double* p : c->erk_k)
    if (p) cudaFree(p);
  if (c->erk_y) cudaFree(c->erk_y);
  for (auto& t : c->tev) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto e : c->pipe_ev) cudaEventDestroy(e);
  if (c->ev_packed) cudaEventDestroy(c->ev_packed);
  if (c->ev_comm) cudaEventDestroy(c->ev_comm);
  if (c->step_graph) cudaGraphExecDestroy(c->step_graph);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

es_status es_setup(es_context** out, const es_mesh* mesh, int p, es_map_fn map, void* user,
                   const es_options* opt) {
  if (!out || !mesh || !opt || !mesh->elem_vertices || !mesh->elem_vertex_coords) return ES_ERR_ARG;
  *out = nullptr;
  es_context* c = new es_context();
  *out = c;
  c->d = mesh->dim;
  c->p = p;
  c->gamma = opt->gamma;
  c->es = opt->interface_flux;
  c->check_adm = opt->check_admissibility;
  c->eq56 = opt->volume_mode == 1;
  c->dense = opt->volume_mode == 2;
  if (opt->volume_mode < 0 || opt->volume_mode > 2) return fail(c, ES_ERR_CONFIG, "volume_mode must be 0, 1 or 2");
  c->rank = opt->rank;
  c->world = opt->world < 1 ? 1 : opt->world;
  c->device = opt->device;
  if (c->d != 2 && c->d != 3) return fail(c, ES_ERR_CONFIG, "dim must be 2 or 3");
  if (!(c->gamma > 1.0)) return fail(c, ES_ERR_CONFIG, "gamma must exceed 1");
  if (c->es < 0 || c->es > 3) return fail(c, ES_ERR_CONFIG, "interface_flux must be 0, 1, 2 or 3");
  if (c->rank < 0 || c->rank >= c->world) return fail(c, ES_ERR_ARG, "rank out of range");
  c->external = c->world > 1 && !opt->nccl_unique_id;
  std::string err;
  if (opt->mapping_nodes != 0 && opt->mapping_nodes != 1) return fail(c, ES_ERR_CONFIG, "mapping_nodes must be 0 or 1");
  if (opt->metric_storage != 0 && opt->metric_storage != 1) return fail(c, ES_ERR_CONFIG, "metric_storage must be 0 or 1");
  c->metric_modal = opt->metric_storage;
  if (!build_ref_tables(c->d, p, c->T, err, opt->mapping_nodes)) return fail(c, ES_ERR_CONFIG, err);
  c->n = c->T.n;
  c->Nq = c->T.Nq;
  c->Nqf = c->T.Nqf;
  c->Nf = c->T.Nf;
  c->Np = c->T.Np;
  c->NC = c->d + 2;
  c->c0 = c->d == 2 ? 1.0 / std::sqrt(2.0) : std::sqrt(0.75);
  // the even-odd psi1 contractions (psi_const.cuh) need psi1[a1][N-1-a] = (-1)^a1 psi1[a1][a]: the
  // Legendre nodes are symmetric and psi1^a1 has the parity of a1 (checked to 2 ulp here)
  for (int a1 = 0; a1 < c->T.n; ++a1)
    for (int a = 0; a < c->T.n; ++a) {
      const double x = c->T.psi1[(size_t)a1 * c->T.n + a], y = c->T.psi1[(size_t)a1 * c->T.n + c->T.n - 1 - a];
      if (std::fabs(x - (a1 % 2 ? -y : y)) > 4.5e-16 * std::fabs(x) + 1e-300)
        return fail(c, ES_ERR_VERIFY, "psi1 table is not parity-symmetric (even-odd transform form)");
    }
  c->ne = mesh->n_elements;
  if (c->ne < c->world) return fail(c, ES_ERR_CONFIG, "fewer elements than ranks");
  if (!build_mesh_plan(c->d, c->ne, mesh->elem_vertices, c->rank, c->world, c->plan, err))
    return fail(c, ES_ERR_VERIFY, err);
  c->first = c->plan.first;
  c->nloc = c->plan.nloc;
  c->nslots = c->nloc * c->Nf + c->plan.n_halo;
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, c->device));
  c->proj_ctas = c->num_sms;  // persistent kernels: SM count x resident CTAs per SM (launcher)
  if (opt->cuda_stream) {
    c->stream = (cudaStream_t)opt->cuda_stream;
  } else {
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
  }
  CK(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_comm, cudaEventDisableTiming));
  es_status s = upload_tables(c);
  if (s != ES_OK) return s;
  if (c->dense) {  // volume_mode 2: dense operators for the brute-force ablation
    std::vector<double> S, RB;
    build_dense_tables(c->T, S, RB);
    CK(cudaMalloc((void**)&c->sdense, S.size() * sizeof(double)));
    CK(cudaMalloc((void**)&c->rbdense, RB.size() * sizeof(double)));
    CK(cudaMemcpy(c->sdense, S.data(), S.size() * sizeof(double), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->rbdense, RB.data(), RB.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  // ---- mapping nodes: affine images of the degree-p lattice, then the user map ----
  const int d = c->d, nv = d + 1, Npg = c->T.Npg;
  std::vector<double> xin((size_t)c->nloc * Npg * d), xmap(xin.size());
  for (int64_t k = 0; k < c->nloc; ++k) {
    const double* X = mesh->elem_vertex_coords + (size_t)(c->first + k) * nv * d;
    for (int i = 0; i < Npg; ++i)
      for (int m = 0; m < d; ++m) {
        double s2 = 0.0;
        for (int v = 0; v < nv; ++v) s2 += c->T.lat_bary[(size_t)i * nv + v] * X[v * d + m];
        xin[((size_t)k * Npg + i) * d + m] = s2;
      }
  }
  if (map)
    map(user, c->nloc * Npg, xin.data(), xmap.data());
  else
    xmap = xin;
  CK(upload(&c->xmapv, xmap));  // absolute mapping-node positions, kept for es_eval_points
  // element-local coordinates (R25): metric terms are translation invariant, and local
  // coordinates avoid a cancellation of order (L/h)^2 in the curl-form metrics
  std::vector<double> shift((size_t)c->nloc * d);
  for (int64_t k = 0; k < c->nloc; ++k)
    for (int m = 0; m < d; ++m) {
      shift[(size_t)k * d + m] = mesh->elem_vertex_coords[(size_t)(c->first + k) * nv * d + m];
      for (int i = 0; i < Npg; ++i) xmap[((size_t)k * Npg + i) * d + m] -= shift[(size_t)k * d + m];
    }
  double* d_shift = nullptr;
  CK(upload(&d_shift, shift));
  // ---- geometry on the device ----
  double* d_xmap = nullptr;
  CK(upload(&d_xmap, xmap));
  const int NG = d * d, NF = c->Nf * c->Nqf;
  CK(cudaMalloc((void**)&c->geo_vol, (size_t)c->nloc * even_up((NG + 2) * c->Nq) * sizeof(double)));
  CK(cudaMalloc((void**)&c->geo_face, (size_t)c->nloc * NF * d * sizeof(double)));
  CK(cudaMalloc((void**)&c->xq, (size_t)c->nloc * c->Nq * d * sizeof(double)));
  CK(cudaMalloc((void**)&c->jt, (size_t)c->nloc * c->Nq * sizeof(double)));
  CK(cudaMalloc((void**)&c->bad, sizeof(int)));
  CK(cudaMemset(c->bad, 0, sizeof(int)));
  std::vector<double*> mats(8, nullptr);
  const std::vector<double>* srcs[8] = {&c->T.LmapV, &c->T.DmapV, &c->T.DmapF, &c->T.DmapM,
                                        &c->T.LmapC, &c->T.DmapC, &c->T.DcurlV, &c->T.DcurlF};
  for (int k = 0; k < 8; ++k) CK(upload(&mats[k], *srcs[k]));
  const double* lo[8];
  for (int k = 0; k < 8; ++k) lo[k] = mats[k] ? mats[k] + srcs[k]->size() / 2 : nullptr;  // [hi | lo]
  GeoArgs g{d, Npg, c->T.Ncl, c->Nq, NF, c->Nqf, even_up((NG + 2) * c->Nq), d_xmap, mats[0], mats[1], mats[2], mats[3], mats[4], mats[5],
            mats[6], mats[7], lo[0], lo[1], lo[2], lo[3], lo[4], lo[5], lo[6], lo[7],
            c->R.Wvol, c->R.nhat, d_shift, c->geo_vol, c->geo_face, c->xq, c->jt, c->bad};
  CK(launch_geometry(g, c->nloc, c->stream));
  c->launches++;
  int hbad = 0;
  CK(cudaMemcpyAsync(&hbad, c->bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d_xmap);
  cudaFree(d_shift);
  for (auto m : mats)
    if (m) cudaFree(m);
  if (hbad) return fail(c, ES_ERR_VERIFY, "non-positive Jacobian (J at a mapping node or J~ at a volume node)");
  // ---- connectivity, lists, face check ----
  CK(upload(&c->face_slot, c->plan.face_slot));
  CK(upload(&c->face_reflect, c->plan.face_reflect));
  CK(upload(&c->d_interior, c->plan.interior));
  CK(upload(&c->d_boundary, c->plan.boundary));
  CK(upload(&c->d_send, c->plan.send_slots));
  unsigned long long* d_mm = nullptr;
  CK(cudaMalloc((void**)&d_mm, sizeof(unsigned long long)));
  CK(cudaMemset(d_mm, 0, sizeof(unsigned long long)));
  FaceCheckArgs fa{d, c->n, c->Nqf, c->nloc, c->geo_face, c->R.Bf, c->face_slot, c->face_reflect, d_mm};
  CK(launch_face_check(fa, c->stream));
  unsigned long long hmm = 0;
  CK(cudaMemcpyAsync(&hmm, d_mm, sizeof(hmm), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(d_mm);
  double mism;
  std::memcpy(&mism, &hmm, sizeof(double));
  if (!(mism < 1e-8))
    return fail(c, ES_ERR_VERIFY, "face normals / weights do not match across faces (rel " + std::to_string(mism) + ")");
  // ---- work buffers ----
  const size_t nmod = (size_t)c->nloc * c->NC * c->Np;
  CK(cudaMalloc((void**)&c->prim, (size_t)c->nloc * even_up((c->NC + 1) * c->Nq + 1) * sizeof(double)));
  CK(cudaMalloc((void**)&c->trace, (size_t)c->nslots * c->NC * c->Nqf * sizeof(double)));
  CK(cudaMalloc((void**)&c->wt, nmod * sizeof(double)));
  CK(cudaMalloc((void**)&c->part, (size_t)c->nloc * (2 + c->NC) * sizeof(double)));
  CK(cudaMalloc((void**)&c->red, 8 * sizeof(double)));
  CK(cudaMalloc((void**)&c->U, nmod * sizeof(double)));
  CK(cudaMalloc((void**)&c->ACC, nmod * sizeof(double)));
  CK(cudaMalloc((void**)&c->US, nmod * sizeof(double)));
  CK(cudaMemset(c->U, 0, nmod * sizeof(double)));
  if (c->d == 3) {  // K3: nodal residual buffer, W / J~ in its layout, PKD tables in constant memory
    CK(cudaMalloc((void**)&c->rbuf, (size_t)c->nloc * c->NC * c->Nq * sizeof(double)));
    CK(cudaMalloc((void**)&c->wjk3, (size_t)c->nloc * c->Nq * sizeof(double)));
    CK(launch_wjinv_permute_3d(c->n, c->geo_vol, even_up((NG + 2) * c->Nq), NG + 1, c->nloc, c->wjk3, c->stream));
    CK(upload_psi_3d(c->n, c->T.psi1.data(), c->T.psi2.data(), c->T.psi3.data()));
    CK(upload_psi_3d_k1(c->n, c->T.psi1.data(), c->T.psi2.data(), c->T.psi3.data()));
    c->launches++;
  }
  if (c->metric_modal) {  // modal metric storage: g~ = V^T W G per element
    const int gms = even_up(NG * c->Np);
    CK(cudaMalloc((void**)&c->gmod, (size_t)c->nloc * gms * sizeof(double)));
    MetricModalArgs mm{d, c->n, c->Nq, c->Np, even_up((NG + 2) * c->Nq), gms, c->nloc, c->geo_vol,
                       c->R.psi1, c->R.psi2, c->R.psi3, c->R.Wvol, c->R.mode_pr, c->R.pair_a1, c->R.pair_a2,
                       c->R.pair_off, c->gmod};
    CK(launch_metric_modal(mm, c->stream));
    c->launches++;
  }
  if (std::getenv("ES_PHASE_TIMING")) {
    CK(cudaMalloc((void**)&c->dbg, 2 * 4096 * 16 * sizeof(long long)));
    CK(cudaMemset(c->dbg, 0, 2 * 4096 * 16 * sizeof(long long)));
  }
  if (c->world > 1) {
    const size_t nsend = c->plan.send_slots.size();
    CK(cudaMalloc((void**)&c->send_buf, std::max<size_t>(nsend, 1) * c->NC * c->Nqf * sizeof(double)));
    if (!c->external) {
      ncclUniqueId id;
      std::memcpy(&id, opt->nccl_unique_id, sizeof(id));
      NK(ncclCommInitRank(&c->comm, c->world, id, c->rank));
    }
  }
  return ES_OK;
}

es_status es_sizes(const es_context* c, int* Np, int* Nq, int* Nqf, int64_t* nloc, int64_t* first) {
  if (!c) return ES_ERR_ARG;
  if (Np) *Np = c->Np;
  if (Nq) *Nq = c->Nq;
  if (Nqf) *Nqf = c->Nqf;
  if (nloc) *nloc = c->nloc;
  if (first) *first = c->first;
  return ES_OK;
}

es_status es_rhs(es_context* c, const double* u, double* dudt) {
  POISON_CHECK();
  if (!u || !dudt) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  RhsArgs A = base_rhs_args(c);
  A.mode = 0;
  A.out = dudt;
  es_status s = rhs_pass(c, u, A, nullptr);
  if (s != ES_OK) return s;
  if (c->dbg) {  // ES_PHASE_TIMING: mean clock cycles per phase over the first blocks of each kernel
    std::vector<long long> h(2 * 4096 * 16);
    CK(cudaStreamSynchronize(c->stream));
    CK(cudaMemcpy(h.data(), c->dbg, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    int nb = (int)std::min<int64_t>(4096, c->nloc);
    for (int kk = 0; kk < 2; ++kk) {
      double acc[16] = {0};
      for (int b = 0; b < nb; ++b)
        for (int k = 1; k < 16; ++k) {
          long long t1 = h[(kk * 4096 + b) * 16 + k], t0 = h[(kk * 4096 + b) * 16 + k - 1];
          if (t1 && t0) acc[k] += (double)(t1 - t0);
        }
      std::fprintf(stderr, "ES_PHASE_TIMING %s cycles/element:", kk ? "project" : "flux");
      for (int k = 1; k < 12; ++k) std::fprintf(stderr, " %d:%.0f", k, acc[k] / nb);
      std::fprintf(stderr, "\n");
    }
  }
  if (c->check_adm) return check_bad(c);
  return ES_OK;
}

es_status es_rhs_host(es_context* c, const double* uh, double* duh) {
  POISON_CHECK();
  if (!uh || !duh) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  const size_t bytes = (size_t)c->nloc * c->NC * c->Np * sizeof(double);
  if (!c->hin) {
    CK(cudaMalloc((void**)&c->hin, bytes));
    CK(cudaMalloc((void**)&c->hout, bytes));
  }
  CK(cudaMemcpyAsync(c->hin, uh, bytes, cudaMemcpyHostToDevice, c->stream));
  es_status s = es_rhs(c, c->hin, c->hout);
  if (s != ES_OK) return s;
  CK(cudaMemcpyAsync(duh, c->hout, bytes, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ES_OK;
}

es_status es_set_state(es_context* c, const double* u) {
  POISON_CHECK();
  c->dp_fsal = false;
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(c->U, u, (size_t)c->nloc * c->NC * c->Np * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return ES_OK;
}
es_status es_get_state(es_context* c, double* u) {
  POISON_CHECK();
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(u, c->U, (size_t)c->nloc * c->NC * c->Np * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return ES_OK;
}

namespace {
// one classical RK4 step (R17): four right-hand sides, the stage update fused in the epilogue
es_status rk4_step_launches(es_context* c, double dt) {
  for (int s = 0; s < 4; ++s) {
    RhsArgs A = base_rhs_args(c);
    A.mode = 1 + s;
    A.dt = dt;
    A.u0 = c->U;
    A.acc = c->ACC;
    A.ustage = c->US;
    A.out = c->U;
    es_status r = rhs_pass(c, s == 0 ? c->U : c->US, A, nullptr);
    if (r != ES_OK) return r;
  }
  return ES_OK;
}
}  // namespace

es_status es_step(es_context* c, double dt, int nsteps) {
  POISON_CHECK();
  c->dp_fsal = false;
  CK(cudaSetDevice(c->device));
  // single rank, no per-kernel timing: the step's launches are captured once into a CUDA graph (per
  // dt, a kernel argument) and replayed -- small meshes are launch-latency bound
  const bool graph = c->use_graphs && c->world == 1 && !c->timing && !c->dbg && nsteps > 0;
  if (graph) {
    if (!c->step_graph || c->step_graph_dt != dt) {
      if (c->step_graph) {
        CK(cudaGraphExecDestroy(c->step_graph));
        c->step_graph = nullptr;
      }
      cudaGraph_t g = nullptr;
      const int64_t l0 = c->launches;
      CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed));
      es_status r = rk4_step_launches(c, dt);
      cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
      if (r != ES_OK) {
        if (g) cudaGraphDestroy(g);
        return r;
      }
      CK(ce);
      ce = cudaGraphInstantiate(&c->step_graph, g, 0);
      cudaGraphDestroy(g);
      CK(ce);
      c->step_graph_dt = dt;
      c->step_graph_launches = c->launches - l0;
      c->launches = l0;
    }
    for (int st = 0; st < nsteps; ++st) {
      CK(cudaGraphLaunch(c->step_graph, c->stream));
      c->launches += c->step_graph_launches;
    }
  } else {
    for (int st = 0; st < nsteps; ++st) {
      es_status r = rk4_step_launches(c, dt);
      if (r != ES_OK) return r;
    }
  }
  if (c->check_adm) return check_bad(c);
  return ES_OK;
}

// es_step_host on one rank, pipelined: the host -> device copy of the state goes in NCH chunks of
// contiguous elements on the copy stream; the first stage's projection K1 runs on each chunk as soon as
// it has arrived (K1 is element-local), and the flux kernel K2 on a chunk as soon as K1 has run on every
// chunk holding a face neighbour of its elements (pipe_dep; with periodic wrap-around the first chunk
// comes last).  In the last stage K2 (+ K3 in 3D) run chunk by chunk and each chunk's device -> host
// copy starts as soon as its new state is written.  Same kernels on the same elements as es_step:
// bitwise equal results (test_step_host_pipelined_bitwise).
namespace {
constexpr int NCH = 8;
es_status step_host_pipelined(es_context* c, const double* u_host, double* u_host_out, double dt, int nsteps) {
  const int64_t per = (int64_t)c->NC * c->Np, n = c->nloc;
  auto lo = [&](int k) { return n * k / NCH; };
  if ((int)c->pipe_ev.size() < 2 * NCH) {
    while ((int)c->pipe_ev.size() < 2 * NCH) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      c->pipe_ev.push_back(e);
    }
    std::vector<int64_t> iota(n);
    for (int64_t e = 0; e < n; ++e) iota[e] = e;
    CK(upload(&c->d_iota, iota));
    c->pipe_dep.assign(NCH, 0);
    for (int k = 0; k < NCH; ++k)
      for (int64_t e = lo(k); e < lo(k + 1); ++e)
        for (int z = 0; z < c->Nf; ++z) {
          const int64_t nb = c->plan.nbr[e * c->Nf + z];
          int kk = 0;
          while (kk + 1 < NCH && lo(kk + 1) <= nb) ++kk;
          c->pipe_dep[k] = std::max(c->pipe_dep[k], std::max(kk, k));
        }
  }
  const int64_t gvs = even_up((c->d * c->d + 2) * c->Nq), prs = even_up((c->NC + 1) * c->Nq + 1),
                trs = (int64_t)c->Nf * c->NC * c->Nqf;
  cudaStream_t cs = c->comm_stream;
  // the copies wait for earlier work on the context stream (which may still use the state)
  CK(cudaEventRecord(c->pipe_ev[0], c->stream));
  CK(cudaStreamWaitEvent(cs, c->pipe_ev[0], 0));
  for (int st = 0; st < nsteps; ++st) {
    for (int s = 0; s < 4; ++s) {
      RhsArgs A = base_rhs_args(c);
      A.mode = 1 + s;
      A.dt = dt;
      A.u0 = c->U;
      A.acc = c->ACC;
      A.ustage = c->US;
      A.out = c->U;
      const bool first = st == 0 && s == 0, last = st == nsteps - 1 && s == 3;
      if (first) {  // chunked H2D -> K1, K2 as soon as the neighbours' traces exist, then K3
        std::vector<char> done(NCH, 0);
        for (int k = 0; k < NCH; ++k) {
          const int64_t e0 = lo(k), ne = lo(k + 1) - e0;
          if (ne > 0) {
            CK(cudaMemcpyAsync(c->U + e0 * per, u_host + e0 * per, (size_t)ne * per * sizeof(double),
                               cudaMemcpyHostToDevice, cs));
            CK(cudaEventRecord(c->pipe_ev[k], cs));
            CK(cudaStreamWaitEvent(c->stream, c->pipe_ev[k], 0));
            ProjArgs P{ne, nullptr, c->U + e0 * per, c->geo_vol + e0 * gvs, c->prim + e0 * prs, c->trace + e0 * trs,
                       nullptr, c->bad, c->gamma, nullptr, c->proj_ctas};
            c->launches++;
            CK(c->d == 2 ? launch_project_2d(c->n, c->R, P, c->stream) : launch_project_3d(c->n, c->R, P, c->stream));
          }
          for (int i = 0; i < NCH; ++i)
            if (!done[i] && c->pipe_dep[i] <= k) {
              CK(run_k2(c, A, lo(i + 1) - lo(i), c->d_iota + lo(i)));
              done[i] = 1;
            }
        }
        CK(run_k3(c, A));
        continue;
      }
      CK(run_project(c, s == 0 ? c->U : c->US, c->nloc, nullptr, nullptr));
      if (!last) {
        CK(run_k2(c, A, c->nloc, nullptr));
        CK(run_k3(c, A));
        continue;
      }
      for (int k = 0; k < NCH; ++k) {  // chunked K2 (+ K3) -> D2H
        const int64_t e0 = lo(k), ne = lo(k + 1) - e0;
        if (ne <= 0) continue;
        CK(run_k2(c, A, ne, c->d_iota + e0));
        if (c->d == 3) {
          WadjArgs W{ne, c->rbuf + e0 * (int64_t)c->NC * c->Nq, c->wjk3 + e0 * (int64_t)c->Nq, A.mode, A.out + e0 * per,
                     A.u0 + e0 * per, A.acc + e0 * per, A.ustage + e0 * per, A.dt, nullptr, nullptr, A.c0};
          c->launches++;
          CK(launch_wadj_3d(c->n, W, c->stream));
        }
        CK(cudaEventRecord(c->pipe_ev[NCH + k], c->stream));
        CK(cudaStreamWaitEvent(cs, c->pipe_ev[NCH + k], 0));
        CK(cudaMemcpyAsync(u_host_out + e0 * per, c->U + e0 * per, (size_t)ne * per * sizeof(double),
                           cudaMemcpyDeviceToHost, cs));
      }
    }
  }
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(cs));
  return ES_OK;
}
}  // namespace

es_status es_step_host(es_context* c, const double* u_host, double* u_host_out, double dt, int nsteps) {
  POISON_CHECK();
  if (!u_host || !u_host_out) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  const size_t bytes = (size_t)c->nloc * c->NC * c->Np * sizeof(double);
  c->dp_fsal = false;
  // large states only (small meshes keep the single CUDA-graph replay of es_step)
  if (c->world == 1 && nsteps >= 1 && !c->timing && !c->dbg && bytes >= ((size_t)64 << 20) && !c->eq56 && !c->dense) {
    es_status s = step_host_pipelined(c, u_host, u_host_out, dt, nsteps);
    if (s != ES_OK) return s;
    if (c->check_adm) return check_bad(c);
    return ES_OK;
  }
  CK(cudaMemcpyAsync(c->U, u_host, bytes, cudaMemcpyHostToDevice, c->stream));
  es_status s = es_step(c, dt, nsteps);
  if (s != ES_OK) return s;
  CK(cudaMemcpyAsync(u_host_out, c->U, bytes, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return ES_OK;
}

es_status es_set_graphs(es_context* c, int on) {
  POISON_CHECK();
  c->use_graphs = on != 0;
  return ES_OK;
}

// Dormand-Prince 5(4) (Hairer-Norsett-Wanner I, Table II.5.2; the paper uses DP8 of the same family,
// P:889).  Stage inputs and the solution are streamed combinations of the slopes (rk_comb_kernel);
// the slopes are full RHS evaluations (mode 0).  FSAL: the last slope f(y5) is the next step's first.
namespace {
const double DPA[7][6] = {{0, 0, 0, 0, 0, 0},
                          {1.0 / 5.0, 0, 0, 0, 0, 0},
                          {3.0 / 40.0, 9.0 / 40.0, 0, 0, 0, 0},
                          {44.0 / 45.0, -56.0 / 15.0, 32.0 / 9.0, 0, 0, 0},
                          {19372.0 / 6561.0, -25360.0 / 2187.0, 64448.0 / 6561.0, -212.0 / 729.0, 0, 0},
                          {9017.0 / 3168.0, -355.0 / 33.0, 46732.0 / 5247.0, 49.0 / 176.0, -5103.0 / 18656.0, 0},
                          {35.0 / 384.0, 0.0, 500.0 / 1113.0, 125.0 / 192.0, -2187.0 / 6784.0, 11.0 / 84.0}};
// b - bh (5th-order weights minus the embedded 4th-order ones)
const double DPE[7] = {35.0 / 384.0 - 5179.0 / 57600.0,     0.0, 500.0 / 1113.0 - 7571.0 / 16695.0,
                       125.0 / 192.0 - 393.0 / 640.0,        -2187.0 / 6784.0 + 92097.0 / 339200.0,
                       11.0 / 84.0 - 187.0 / 2100.0,         -1.0 / 40.0};
}  // namespace

es_status es_step_dp54(es_context* c, double dt, double rtol, double atol, double* err, int* accepted) {
  POISON_CHECK();
  if (!err || !accepted || !(dt > 0.0) || !(rtol >= 0.0) || !(atol >= 0.0) || !(rtol > 0.0 || atol > 0.0))
    return fail(c, ES_ERR_ARG, "es_step_dp54: dt > 0, rtol, atol >= 0 (not both 0), err and accepted required");
  CK(cudaSetDevice(c->device));
  const int64_t n = c->nloc * (int64_t)c->NC * c->Np;
  if (!c->dpy) {
    for (auto& p : c->dpk) CK(cudaMalloc((void**)&p, (size_t)n * sizeof(double)));
    CK(cudaMalloc((void**)&c->dpy, (size_t)n * sizeof(double)));
    CK(cudaMalloc((void**)&c->dppart, RK_ERR_BLOCKS * sizeof(double)));
    c->dp_fsal = false;
  }
  auto slope = [&](const double* y, double* k) -> es_status {
    RhsArgs A = base_rhs_args(c);
    A.mode = 0;
    A.out = k;
    return rhs_pass(c, y, A, nullptr);
  };
  es_status r;
  if (!c->dp_fsal && (r = slope(c->U, c->dpk[0])) != ES_OK) return r;
  for (int st = 1; st < 7; ++st) {
    RkComb kc{};
    kc.nk = st;
    for (int j = 0; j < st; ++j) {
      kc.k[j] = c->dpk[j];
      kc.c[j] = dt * DPA[st][j];
    }
    double* ys = st == 6 ? c->dpy : c->US;  // the last stage input is the 5th-order solution
    CK(launch_rk_comb(c->U, kc, ys, n, c->stream));
    c->launches++;
    if ((r = slope(ys, c->dpk[st])) != ES_OK) return r;
  }
  RkComb ec{};
  ec.nk = 7;
  for (int j = 0; j < 7; ++j) {
    ec.k[j] = c->dpk[j];
    ec.c[j] = dt * DPE[j];
  }
  CK(launch_rk_err(c->U, c->dpy, ec, rtol, atol, n, c->dppart, c->stream));
  CK(launch_reduce_parts(c->dppart, RK_ERR_BLOCKS, 1, c->red, c->stream));
  c->launches += 2;
  double hsum[2] = {0.0, (double)n};
  CK(cudaMemcpyAsync(hsum, c->red, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->world > 1) {
    if (!c->comm) return fail(c, ES_ERR_CONFIG, "es_step_dp54 with world > 1 needs the NCCL communicator");
    double* d2 = c->red;
    CK(cudaMemcpyAsync(d2, hsum, 2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    NK(ncclAllReduce(d2, d2, 2, ncclDouble, ncclSum, c->comm, c->stream));
    CK(cudaMemcpyAsync(hsum, d2, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  *err = sqrt(hsum[0] / hsum[1]);
  *accepted = *err <= 1.0;
  if (*accepted) {  // y5 becomes the state, f(y5) the next first slope
    std::swap(c->U, c->dpy);
    std::swap(c->dpk[0], c->dpk[6]);
    c->dp_fsal = true;
  } else {
    c->dp_fsal = true;  // dpk[0] = f(U) still holds
  }
  if (c->check_adm) return check_bad(c);
  return ES_OK;
}

es_status es_step_erk(es_context* c, double dt, int s, const double* A, const double* b, int nsteps) {
  POISON_CHECK();
  if (!A || !b || s < 1 || s > 16 || !(dt > 0.0))
    return fail(c, ES_ERR_ARG, "es_step_erk: 1 <= s <= 16 stages, A[s][s], b[s], dt > 0");
  for (int i = 0; i < s; ++i)
    for (int j = i; j < s; ++j)
      if (A[i * s + j] != 0.0) return fail(c, ES_ERR_ARG, "es_step_erk: A must be strictly lower triangular");
  CK(cudaSetDevice(c->device));
  c->dp_fsal = false;
  const int64_t n = c->nloc * (int64_t)c->NC * c->Np;
  while ((int)c->erk_k.size() < s) {
    double* p = nullptr;
    CK(cudaMalloc((void**)&p, (size_t)n * sizeof(double)));
    c->erk_k.push_back(p);
  }
  if (!c->erk_y) CK(cudaMalloc((void**)&c->erk_y, (size_t)n * sizeof(double)));
  for (int st = 0; st < nsteps; ++st) {
    for (int i = 0; i < s; ++i) {  // k_i = f(U + dt sum_{l<i} a_il k_l)
      const double* y = c->U;
      RkComb kc{};
      for (int l = 0; l < i; ++l)
        if (A[i * s + l] != 0.0) {
          kc.k[kc.nk] = c->erk_k[l];
          kc.c[kc.nk++] = dt * A[i * s + l];
        }
      if (kc.nk > 0) {
        CK(launch_rk_comb(c->U, kc, c->US, n, c->stream));
        c->launches++;
        y = c->US;
      }
      RhsArgs Ar = base_rhs_args(c);
      Ar.mode = 0;
      Ar.out = c->erk_k[i];
      es_status r = rhs_pass(c, y, Ar, nullptr);
      if (r != ES_OK) return r;
    }
    RkComb kc{};
    for (int l = 0; l < s; ++l)
      if (b[l] != 0.0) {
        kc.k[kc.nk] = c->erk_k[l];
        kc.c[kc.nk++] = dt * b[l];
      }
    CK(launch_rk_comb(c->U, kc, c->erk_y, n, c->stream));
    c->launches++;
    std::swap(c->U, c->erk_y);
  }
  if (c->check_adm) return check_bad(c);
  return ES_OK;
}

es_status es_entropy_production(es_context* c, const double* u, double* rate, double* abs_scale,
                                 double* cons) {
  POISON_CHECK();
  CK(cudaSetDevice(c->device));
  // a flag left by an earlier unchecked call (check_admissibility = 0) must not be reported here
  CK(cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream));
  double* scratch = c->ACC;  // the RK accumulator is free between steps
  RhsArgs A = base_rhs_args(c);
  A.mode = 5;
  A.out = scratch;
  A.wt = c->wt;
  A.part = c->part;
  es_status s = rhs_pass(c, u, A, c->wt);
  if (s != ES_OK) return s;
  const int w = 2 + c->NC;
  CK(launch_reduce_parts(c->part, c->nloc, w, c->red, c->stream));
  c->launches++;
  if (c->world > 1 && c->comm) NK(ncclAllReduce(c->red, c->red, w, ncclDouble, ncclSum, c->comm, c->stream));
  double h[8] = {0};
  CK(cudaMemcpyAsync(h, c->red, w * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (rate) *rate = h[0];
  if (abs_scale) *abs_scale = h[1];
  if (cons)
    for (int v = 0; v < c->NC; ++v) cons[v] = h[2 + v];
  return check_bad(c);
}

es_status es_flux_counts(const es_context* c, int64_t* vol, int64_t* fac, int64_t* eq56, double* iface) {
  if (!c) return ES_ERR_ARG;
  int64_t n = c->n, q = c->p;
  if (c->d == 2) {
    // line-wise: one flux per pair on each eta line, n(n-1)/2 pairs per line, n lines per direction;
    // Eq. num_fluxes mode: one per operator with a nonzero on the line (2 on eta1, 1 on eta2 lines)
    if (vol) *vol = c->dense ? n * n * (n * n - 1) : c->eq56 ? 3 * q * n * n / 2 : q * n * n;
    if (fac) *fac = c->dense ? 2 * (n * n) * (3 * n)  // every (node, facet node) pair, from both sides
                             : 3 * n * n;             // n volume nodes per facet node, 3 facets
    if (eq56) *eq56 = 3 * n * n * (q + 2) / 2; // sum_l nnz(S^(l))/2 + sum nnz(R^T B)
    if (iface) *iface = 3.0 * n;               // per element side
  } else {
    if (vol) *vol = c->dense ? n * n * n * (n * n * n - 1)  // brute force: every ordered pair
                             : c->eq56 ? 3 * q * n * n * n : 3 * q * n * n * n / 2;  // (3 + 2 + 1) vs 3 line directions
    if (fac) *fac = c->dense ? 2 * (n * n * n) * (4 * n * n) : 3 * n * n * n + n * n * n * n;
    if (eq56) *eq56 = 4 * n * n * n * n;
    if (iface) *iface = 4.0 * n * n;
  }
  return ES_OK;
}

es_status es_count_fluxes(es_context* c, const double* u, int64_t* counts) {
  POISON_CHECK();
  if (!u || !counts) return fail(c, ES_ERR_ARG, "null buffer");
  if (c->dense) return fail(c, ES_ERR_CONFIG, "es_count_fluxes: volume_mode 2 is not instrumented");
  CK(cudaSetDevice(c->device));
  const size_t nb = (size_t)c->nloc * 4 * sizeof(unsigned long long);
  if (!c->dcounts) CK(cudaMalloc((void**)&c->dcounts, nb));
  CK(cudaMemsetAsync(c->dcounts, 0, nb, c->stream));
  RhsArgs A = base_rhs_args(c);
  A.mode = 0;
  A.out = c->ACC;  // scratch: the RK accumulator is free between steps
  c->counting = true;
  es_status s = rhs_pass(c, u, A, nullptr);
  c->counting = false;
  if (s != ES_OK) return s;
  std::vector<unsigned long long> h((size_t)c->nloc * 4);
  CK(cudaMemcpyAsync(h.data(), c->dcounts, nb, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  for (size_t k = 0; k < h.size(); ++k) counts[k] = (int64_t)h[k];
  return ES_OK;
}

es_status es_eval_points(es_context* c, const double* u, int npts, const double* xi, double* uo, double* xo,
                         double* jo) {
  POISON_CHECK();
  if (!u || !xi || !uo || npts <= 0) return fail(c, ES_ERR_ARG, "es_eval_points: u, xi, u_out and npts > 0 required");
  CK(cudaSetDevice(c->device));
  std::vector<double> pkd, lm, dm;
  if (!eval_point_tables(c->d, c->p, xi, npts, pkd, lm, dm, c->T.nodes)) return fail(c, ES_ERR_CONFIG, "point tables");
  double *dp = nullptr, *dl = nullptr, *dd = nullptr;
  CK(upload(&dp, pkd));
  CK(upload(&dl, lm));
  CK(upload(&dd, dm));
  EvalPtsArgs a{c->d, c->NC, c->Np, c->T.Npg, npts, c->nloc, u, c->xmapv, dp, dl, dd, uo, xo, jo};
  CK(launch_eval_points(a, c->stream));
  c->launches++;
  CK(cudaStreamSynchronize(c->stream));
  cudaFree(dp);
  cudaFree(dl);
  cudaFree(dd);
  return ES_OK;
}

// ---- linear advection, single rank ----
es_status es_adv_configure(es_context* c, const double* a, int flux_mode, int form) {
  POISON_CHECK();
  if (!a || flux_mode < 0 || flux_mode > 1 || form < 0 || form > 1)
    return fail(c, ES_ERR_ARG, "es_adv_configure: velocity, flux_mode 0/1, form 0/1");
  if (c->world != 1) return fail(c, ES_ERR_CONFIG, "es_adv_*: single rank only");
  CK(cudaSetDevice(c->device));
  for (int m = 0; m < 3; ++m) c->adv_a[m] = m < c->d ? a[m] : 0.0;
  c->adv_flux = flux_mode;
  c->adv_form = form;
  if (!c->adv_unod) {
    const int n = c->n;
    CK(cudaMalloc((void**)&c->adv_unod, (size_t)c->nloc * c->Nq * sizeof(double)));
    CK(cudaMalloc((void**)&c->adv_trace, (size_t)c->nloc * c->Nf * c->Nqf * sizeof(double)));
    CK(cudaMalloc((void**)&c->adv_acc, (size_t)c->nloc * c->Np * sizeof(double)));
    CK(cudaMalloc((void**)&c->adv_us, (size_t)c->nloc * c->Np * sizeof(double)));
    CK(cudaMalloc((void**)&c->adv_part, (size_t)c->nloc * 2 * sizeof(double)));
    std::vector<double> X((size_t)5 * n * n, 0.0);
    const std::vector<double>* src[5] = {&c->T.fQ1, &c->T.fA1, &c->T.fA2, &c->T.fA3, &c->T.fA4};
    for (int k = 0; k < 5; ++k)
      if (!src[k]->empty()) std::memcpy(&X[(size_t)k * n * n], src[k]->data(), (size_t)n * n * sizeof(double));
    CK(upload(&c->adv_X, X));
    if (c->d == 3) CK(upload_psi_adv_3d(c->n, c->T.psi1.data(), c->T.psi2.data(), c->T.psi3.data()));
  }
  c->adv_ready = true;
  return ES_OK;
}

namespace {
AdvArgs adv_args(es_context* c, const double* u, int mode) {
  AdvArgs A{};
  A.n_elem = c->nloc;
  A.u = u;
  A.unod = c->adv_unod;
  A.trace = c->adv_trace;
  A.geo_vol = c->geo_vol;
  A.geo_face = c->geo_face;
  A.face_slot = c->face_slot;
  A.face_reflect = c->face_reflect;
  A.X = c->adv_X;
  for (int m = 0; m < 3; ++m) A.a[m] = c->adv_a[m];
  A.flux_mode = c->adv_flux;
  A.form = c->adv_form;
  A.mode = mode;
  return A;
}
cudaError_t adv_launch(es_context* c, const AdvArgs& A) {
  c->launches += 2;
  return c->d == 2 ? launch_adv_2d(c->n, c->R, A, c->stream) : launch_adv_3d(c->n, c->R, A, c->stream);
}
}  // namespace

es_status es_adv_rhs(es_context* c, const double* u, double* dudt, double* energy) {
  POISON_CHECK();
  if (!c->adv_ready) return fail(c, ES_ERR_CONFIG, "es_adv_rhs: call es_adv_configure first");
  if (!u || !dudt) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  AdvArgs A = adv_args(c, u, 0);
  A.out = dudt;
  A.part = energy ? c->adv_part : nullptr;
  CK(adv_launch(c, A));
  if (energy) {
    CK(launch_reduce_parts(c->adv_part, c->nloc, 2, c->red, c->stream));
    c->launches++;
    CK(cudaMemcpyAsync(energy, c->red, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  }
  return ES_OK;
}

es_status es_adv_step(es_context* c, double* u, double dt, int nsteps) {
  POISON_CHECK();
  if (!c->adv_ready) return fail(c, ES_ERR_CONFIG, "es_adv_step: call es_adv_configure first");
  if (!u) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  for (int st = 0; st < nsteps; ++st)
    for (int s = 0; s < 4; ++s) {  // classical RK4 (R17), the stage update fused in the epilogue
      AdvArgs A = adv_args(c, s == 0 ? u : c->adv_us, 1 + s);
      A.dt = dt;
      A.u0 = u;
      A.acc = c->adv_acc;
      A.ustage = c->adv_us;
      A.out = u;
      CK(adv_launch(c, A));
    }
  return ES_OK;
}

es_status es_node_coords(es_context* c, double* x) {
  POISON_CHECK();
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(x, c->xq, (size_t)c->nloc * c->Nq * c->d * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return ES_OK;
}

es_status es_project_nodal(es_context* c, const double* un, double* um) {
  POISON_CHECK();
  CK(cudaSetDevice(c->device));
  c->launches++;
  CK(c->d == 2 ? launch_projnodal_2d(c->n, c->R, c->nloc, un, um, c->stream)
               : launch_projnodal_3d(c->n, c->R, c->nloc, un, um, c->stream));
  return ES_OK;
}

es_status es_eval_nodal(es_context* c, const double* um, double* un) {
  POISON_CHECK();
  if (!um || !un) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  c->launches++;
  CK(c->d == 2 ? launch_evalnodal_2d(c->n, c->R, c->nloc, um, un, c->stream)
               : launch_evalnodal_3d(c->n, c->R, c->nloc, um, un, c->stream));
  return ES_OK;
}

es_status es_node_weights(es_context* c, double* wj) {
  POISON_CHECK();
  if (!wj) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  const int NG = c->d * c->d, gvs = even_up((NG + 2) * c->Nq);
  CK(cudaMemcpy2DAsync(wj, (size_t)c->Nq * sizeof(double), c->geo_vol + (size_t)NG * c->Nq, (size_t)gvs * sizeof(double),
                       (size_t)c->Nq * sizeof(double), (size_t)c->nloc, cudaMemcpyDeviceToDevice, c->stream));
  return ES_OK;
}

es_status es_element_geometry(es_context* c, int64_t k, double* G, double* Jn, double* Jt) {
  POISON_CHECK();
  if (k < 0 || k >= c->nloc) return fail(c, ES_ERR_ARG, "element out of range");
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  const int d = c->d, NG = d * d, Nq = c->Nq, Nqf = c->Nqf, Nf = c->Nf;
  if (G) {
    std::vector<double> gv((size_t)NG * Nq);
    CK(cudaMemcpy(gv.data(), c->geo_vol + (size_t)k * even_up((NG + 2) * Nq), gv.size() * 8, cudaMemcpyDeviceToHost));
    for (int i = 0; i < Nq; ++i)
      for (int q = 0; q < NG; ++q) G[(size_t)i * NG + q] = gv[(size_t)q * Nq + i];
  }
  if (Jn) {
    std::vector<double> gf((size_t)Nf * d * Nqf);
    CK(cudaMemcpy(gf.data(), c->geo_face + (size_t)k * Nf * d * Nqf, gf.size() * 8, cudaMemcpyDeviceToHost));
    for (int z = 0; z < Nf; ++z)
      for (int f = 0; f < Nqf; ++f)
        for (int m = 0; m < d; ++m) Jn[((size_t)z * Nqf + f) * d + m] = gf[((size_t)z * d + m) * Nqf + f];
  }
  if (Jt) CK(cudaMemcpy(Jt, c->jt + (size_t)k * Nq, (size_t)Nq * 8, cudaMemcpyDeviceToHost));
  return ES_OK;
}

es_status es_ref_table(int dim, int p, const char* name, double* out, int64_t cap, int64_t* n) {
  if (!name) return ES_ERR_ARG;
  RefTables t;
  std::string err;
  if (!std::strcmp(name, "nodes0") || !std::strcmp(name, "nodes1")) {  // mapping-node barycentrics of degree p
    if ((dim != 2 && dim != 3) || p < 1 || p > 12) return ES_ERR_ARG;
    const std::vector<double> b = node_family_bary(dim, p, name[5] - '0');
    if (n) *n = (int64_t)b.size();
    if (out) {
      if (cap < (int64_t)b.size()) return ES_ERR_ARG;
      std::memcpy(out, b.data(), b.size() * sizeof(double));
    }
    return ES_OK;
  }
  if (!build_ref_tables(dim, p, t, err)) return ES_ERR_CONFIG;
  std::string nm(name);
  const std::vector<double>* v = nullptr;
  if (nm == "eta") v = &t.eta;
  else if (nm == "w") v = &t.w;
  else if (nm == "eta3") v = &t.eta3;
  else if (nm == "w3") v = &t.w3;
  else if (nm == "skQ1") v = &t.skQ1;
  else if (nm == "skA1") v = &t.skA1;
  else if (nm == "skA2") v = &t.skA2;
  else if (nm == "skA3") v = &t.skA3;
  else if (nm == "skA4") v = &t.skA4;
  else if (nm == "fQ1") v = &t.fQ1;
  else if (nm == "fA1") v = &t.fA1;
  else if (nm == "fA2") v = &t.fA2;
  else if (nm == "fA3") v = &t.fA3;
  else if (nm == "fA4") v = &t.fA4;
  else if (nm == "lL") v = &t.lL;
  else if (nm == "lR") v = &t.lR;
  else if (nm == "l3L") v = &t.l3L;
  else if (nm == "lint4") v = &t.lint4;
  else if (nm == "psi1") v = &t.psi1;
  else if (nm == "psi2") v = &t.psi2;
  else if (nm == "psi3") v = &t.psi3;
  else if (nm == "Wvol") v = &t.Wvol;
  else if (nm == "Bf") v = &t.Bf;
  else if (nm == "xi_vol") v = &t.xi_vol;
  if (!v) return ES_ERR_ARG;
  if (n) *n = (int64_t)v->size();
  if (out) {
    if (cap < (int64_t)v->size()) return ES_ERR_ARG;
    std::memcpy(out, v->data(), v->size() * sizeof(double));
  }
  return ES_OK;
}

es_status es_plan(int dim, int64_t ne, const int64_t* ev, int rank, int world, int64_t* face_slot,
                  int* face_reflect, int64_t* send_slots, int64_t* send_count, int64_t* recv_count,
                  int64_t* n_send, int64_t* n_halo) {
  if (!ev || world < 1 || rank < 0 || rank >= world || (dim != 2 && dim != 3)) return ES_ERR_ARG;
  MeshPlan plan;
  std::string err;
  if (!build_mesh_plan(dim, ne, ev, rank, world, plan, err)) return ES_ERR_VERIFY;
  if (face_slot) std::memcpy(face_slot, plan.face_slot.data(), plan.face_slot.size() * sizeof(int64_t));
  if (face_reflect) std::memcpy(face_reflect, plan.face_reflect.data(), plan.face_reflect.size() * sizeof(int));
  if (send_slots) std::memcpy(send_slots, plan.send_slots.data(), plan.send_slots.size() * sizeof(int64_t));
  if (send_count) std::memcpy(send_count, plan.send_count.data(), plan.send_count.size() * sizeof(int64_t));
  if (recv_count) std::memcpy(recv_count, plan.recv_count.data(), plan.recv_count.size() * sizeof(int64_t));
  if (n_send) *n_send = (int64_t)plan.send_slots.size();
  if (n_halo) *n_halo = plan.n_halo;
  return ES_OK;
}

es_status es_rhs_stage1(es_context* c, const double* u, double** send_buf) {
  POISON_CHECK();
  if (!u) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  es_status s = rhs_first(c, u, nullptr);
  if (s != ES_OK) return s;
  if (send_buf) *send_buf = c->send_buf;
  return ES_OK;
}

es_status es_halo_buffer(es_context* c, double** recv_buf) {
  POISON_CHECK();
  if (recv_buf) *recv_buf = c->trace + (size_t)c->nloc * c->Nf * c->NC * c->Nqf;
  return ES_OK;
}

es_status es_rhs_stage2(es_context* c, double* dudt) {
  POISON_CHECK();
  if (!dudt) return fail(c, ES_ERR_ARG, "null buffer");
  CK(cudaSetDevice(c->device));
  RhsArgs A = base_rhs_args(c);
  A.mode = 0;
  A.out = dudt;
  es_status s = rhs_second(c, A);
  if (s != ES_OK) return s;
  if (c->check_adm) return check_bad(c);
  return ES_OK;
}

}  // extern "C"
namespace {
// a loopback group: world contexts of one mesh (ranks 0..world-1, each created without an NCCL id)
// on one device in this process
es_status group_check(es_context** g, int n) {
  if (!g || n < 1) return ES_ERR_ARG;
  for (int r = 0; r < n; ++r) {
    es_context* c = g[r];
    if (!c) return ES_ERR_ARG;
    if (c->poisoned != ES_OK) return c->poisoned;
    if (c->world != n || c->rank != r || c->device != g[0]->device || c->ne != g[0]->ne || c->p != g[0]->p)
      return fail(c, ES_ERR_ARG, "es_group_*: contexts must be ranks 0..n-1 of one mesh on one device");
  }
  return ES_OK;
}
// one RHS of every context of the group with argument builder `args(r)`; the packs of round k wait
// for every receiver's copies of round k-1 (the send buffers are reused)
template <class F>
es_status group_rhs_pass(es_context** g, int n, const double* const* u, F args, double* const* wt) {
  for (int r = 0; r < n; ++r) {
    es_context* c = g[r];
    for (int q = 0; q < n; ++q)
      if (q != r && n > 1) {
        cudaError_t e = cudaStreamWaitEvent(c->stream, g[q]->ev_comm, 0);
        if (e != cudaSuccess) return fail(c, ES_ERR_CUDA, std::string("cudaStreamWaitEvent: ") + cudaGetErrorString(e));
      }
    es_status s = rhs_phase_a(c, u[r], wt ? wt[r] : nullptr);
    if (s != ES_OK) return s;
  }
  for (int r = 0; r < n && n > 1; ++r) {
    es_status s = rhs_phase_b_loopback(g[r], g);
    if (s != ES_OK) return s;
  }
  for (int r = 0; r < n; ++r) {
    es_status s = rhs_phase_c(g[r], args(r));
    if (s != ES_OK) return s;
  }
  return ES_OK;
}
}  // namespace
extern "C" {

es_status es_group_rhs(es_context** g, int n, const double* const* u, double* const* dudt) {
  es_status s = group_check(g, n);
  if (s != ES_OK) return s;
  if (!u || !dudt) return ES_ERR_ARG;
  return group_rhs_pass(g, n, u, [&](int r) {
    RhsArgs A = base_rhs_args(g[r]);
    A.mode = 0;
    A.out = dudt[r];
    return A;
  }, nullptr);
}

es_status es_group_step(es_context** g, int n, double dt, int nsteps) {
  es_status s = group_check(g, n);
  if (s != ES_OK) return s;
  std::vector<const double*> u0(n), us(n);
  for (int r = 0; r < n; ++r) {
    g[r]->dp_fsal = false;
    u0[r] = g[r]->U;
    us[r] = g[r]->US;
  }
  for (int st = 0; st < nsteps; ++st)
    for (int k = 0; k < 4; ++k) {  // classical RK4 (R17), the stage update fused in the epilogue
      s = group_rhs_pass(g, n, k == 0 ? u0.data() : us.data(), [&](int r) {
        es_context* c = g[r];
        RhsArgs A = base_rhs_args(c);
        A.mode = 1 + k;
        A.dt = dt;
        A.u0 = c->U;
        A.acc = c->ACC;
        A.ustage = c->US;
        A.out = c->U;
        return A;
      }, nullptr);
      if (s != ES_OK) return s;
    }
  for (int r = 0; r < n; ++r)
    if (g[r]->check_adm && (s = check_bad(g[r])) != ES_OK) return s;
  return ES_OK;
}

es_status es_group_entropy_production(es_context** g, int n, const double* const* u, double* rate, double* abs_scale,
                                      double* cons) {
  es_status s = group_check(g, n);
  if (s != ES_OK) return s;
  if (!u) return ES_ERR_ARG;
  std::vector<double*> wts(n);
  for (int r = 0; r < n; ++r) {
    es_context* c = g[r];
    cudaError_t e = cudaMemsetAsync(c->bad, 0, sizeof(int), c->stream);
    if (e != cudaSuccess) return fail(c, ES_ERR_CUDA, cudaGetErrorString(e));
    wts[r] = c->wt;
  }
  s = group_rhs_pass(g, n, u, [&](int r) {
    es_context* c = g[r];
    RhsArgs A = base_rhs_args(c);
    A.mode = 5;
    A.out = c->ACC;
    A.wt = c->wt;
    A.part = c->part;
    return A;
  }, wts.data());
  if (s != ES_OK) return s;
  // per-rank deterministic reductions, then the sum over ranks in rank order (the allreduce of
  // es_entropy_production)
  double tot[8] = {0};
  for (int r = 0; r < n; ++r) {
    es_context* c = g[r];
    const int w = 2 + c->NC;
    CK(launch_reduce_parts(c->part, c->nloc, w, c->red, c->stream));
    c->launches++;
    double h[8] = {0};
    CK(cudaMemcpyAsync(h, c->red, w * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < w; ++k) tot[k] += h[k];
    if ((s = check_bad(c)) != ES_OK) return s;
  }
  if (rate) *rate = tot[0];
  if (abs_scale) *abs_scale = tot[1];
  if (cons)
    for (int v = 0; v < g[0]->NC; ++v) cons[v] = tot[2 + v];
  return ES_OK;
}

es_status es_synchronize(es_context* c) {
  POISON_CHECK();
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaGetLastError());
  return ES_OK;
}

void* es_stream(const es_context* c) { return c ? (void*)c->stream : nullptr; }
int64_t es_launch_count(const es_context* c) { return c ? c->launches : 0; }
void es_reset_launch_count(es_context* c) {
  if (c) c->launches = 0;
}

es_status es_timing_enable(es_context* c, int on) {
  POISON_CHECK();
  CK(cudaStreamSynchronize(c->stream));
  for (auto& t : c->tev) {
    c->ev_pool.push_back(t.a);
    c->ev_pool.push_back(t.b);
  }
  c->tev.clear();
  c->timing = on != 0;
  return ES_OK;
}

es_status es_timing_read(es_context* c, int cls, double* total_ms, int64_t* launches) {
  POISON_CHECK();
  CK(cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  int64_t cnt = 0;
  for (auto& t : c->tev) {
    if (t.cls != cls) continue;
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    tot += ms;
    ++cnt;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = cnt;
  return ES_OK;
}

}  // extern "C"
