"""Python binding of the B200-native ES modal DSEM library (include/es.h).

Argument marshalling only: every step of the right-hand side runs in the sm_100a kernels of
libes_b200.so.  There is no CPU fallback -- importing this package fails loudly when the CUDA
library is missing.  PyTorch is used by callers for device memory and streams; this module only
passes raw pointers.
"""
from __future__ import annotations

import ctypes
import math
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libes_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "es.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)
_dp = ctypes.POINTER(ctypes.c_double)
_lp = ctypes.POINTER(ctypes.c_int64)
_vp = ctypes.c_void_p

ES_OK, ES_ERR_CONFIG, ES_ERR_INADMISSIBLE, ES_ERR_VERIFY = 0, 2, 3, 4
ES_ERR_ARG, ES_ERR_CUDA, ES_ERR_NCCL, ES_ERR_OOM = -1, -5, -6, -7

es_map_fn = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, _dp, _dp)


class es_mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("n_elements", ctypes.c_int64), ("elem_vertices", _lp),
                ("elem_vertex_coords", _dp), ("period", _dp)]


class es_options(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("interface_flux", ctypes.c_int), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("nccl_unique_id", ctypes.c_char_p), ("cuda_stream", _vp),
                ("device", ctypes.c_int), ("check_admissibility", ctypes.c_int), ("volume_mode", ctypes.c_int),
                ("mapping_nodes", ctypes.c_int), ("metric_storage", ctypes.c_int)]


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_i = ctypes.c_int
es_setup = _sig("es_setup", _i, ctypes.POINTER(_vp), ctypes.POINTER(es_mesh), _i, es_map_fn, _vp,
                ctypes.POINTER(es_options))
es_destroy = _sig("es_destroy", None, _vp)
es_last_error = _sig("es_last_error", ctypes.c_char_p, _vp)
es_sizes = _sig("es_sizes", _i, _vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i),
                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64))
es_rhs = _sig("es_rhs", _i, _vp, _vp, _vp)
es_rhs_host = _sig("es_rhs_host", _i, _vp, _vp, _vp)
es_set_state = _sig("es_set_state", _i, _vp, _vp)
es_get_state = _sig("es_get_state", _i, _vp, _vp)
es_step = _sig("es_step", _i, _vp, ctypes.c_double, _i)
es_step_dp54 = _sig("es_step_dp54", _i, _vp, ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp,
                    ctypes.POINTER(_i))
es_entropy_production = _sig("es_entropy_production", _i, _vp, _vp, _dp, _dp, _dp)
es_flux_counts = _sig("es_flux_counts", _i, _vp, _lp, _lp, _lp, _dp)
es_count_fluxes = _sig("es_count_fluxes", _i, _vp, _vp, _lp)
es_step_host = _sig("es_step_host", _i, _vp, _vp, _vp, ctypes.c_double, _i)
es_set_graphs = _sig("es_set_graphs", _i, _vp, _i)
es_eval_points = _sig("es_eval_points", _i, _vp, _vp, _i, _dp, _vp, _vp, _vp)
es_step_erk = _sig("es_step_erk", _i, _vp, ctypes.c_double, _i, _dp, _dp, _i)
es_adv_configure = _sig("es_adv_configure", _i, _vp, _dp, _i, _i)
es_adv_rhs = _sig("es_adv_rhs", _i, _vp, _vp, _vp, _dp)
es_adv_step = _sig("es_adv_step", _i, _vp, _vp, ctypes.c_double, _i)
es_group_rhs = _sig("es_group_rhs", _i, ctypes.POINTER(_vp), _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp))
es_group_step = _sig("es_group_step", _i, ctypes.POINTER(_vp), _i, ctypes.c_double, _i)
es_group_entropy_production = _sig("es_group_entropy_production", _i, ctypes.POINTER(_vp), _i, ctypes.POINTER(_vp),
                                   _dp, _dp, _dp)
es_node_coords = _sig("es_node_coords", _i, _vp, _vp)
es_project_nodal = _sig("es_project_nodal", _i, _vp, _vp, _vp)
es_eval_nodal = _sig("es_eval_nodal", _i, _vp, _vp, _vp)
es_node_weights = _sig("es_node_weights", _i, _vp, _vp)
es_element_geometry = _sig("es_element_geometry", _i, _vp, ctypes.c_int64, _dp, _dp, _dp)
es_synchronize = _sig("es_synchronize", _i, _vp)
es_rhs_stage1 = _sig("es_rhs_stage1", _i, _vp, _vp, ctypes.POINTER(_vp))
es_halo_buffer = _sig("es_halo_buffer", _i, _vp, ctypes.POINTER(_vp))
es_rhs_stage2 = _sig("es_rhs_stage2", _i, _vp, _vp)
es_stream = _sig("es_stream", _vp, _vp)
es_launch_count = _sig("es_launch_count", ctypes.c_int64, _vp)
es_reset_launch_count = _sig("es_reset_launch_count", None, _vp)
es_timing_enable = _sig("es_timing_enable", _i, _vp, _i)
es_timing_read = _sig("es_timing_read", _i, _vp, _i, _dp, _lp)
es_ref_table = _sig("es_ref_table", _i, _i, _i, ctypes.c_char_p, _dp, ctypes.c_int64, _lp)
_ip = ctypes.POINTER(ctypes.c_int)
es_plan = _sig("es_plan", _i, _i, ctypes.c_int64, _lp, _i, _i, _lp, _ip, _lp, _lp, _lp, _lp, _lp)


def ref_table(dim, p, name):
    """Host-only copy of one reference table the kernels use (see es_ref_table)."""
    n = ctypes.c_int64()
    rc = es_ref_table(dim, p, name.encode(), None, 0, ctypes.byref(n))
    if rc != ES_OK:
        raise ESError(rc, f"unknown table {name}")
    out = np.zeros(n.value)
    rc = es_ref_table(dim, p, name.encode(), out.ctypes.data_as(_dp), n.value, ctypes.byref(n))
    if rc != ES_OK:
        raise ESError(rc, name)
    return out


def plan(dim, elem_vertices, rank, world):
    """Host-only connectivity / halo plan of one rank (see es_plan)."""
    ev = np.ascontiguousarray(elem_vertices, dtype=np.int64)
    ne = len(ev)
    nf = dim + 1
    first, nloc = ne * rank // world, ne * (rank + 1) // world - ne * rank // world
    ns, nh = ctypes.c_int64(), ctypes.c_int64()
    rc = es_plan(dim, ne, ev.ctypes.data_as(_lp), rank, world, None, None, None, None, None,
                 ctypes.byref(ns), ctypes.byref(nh))
    if rc != ES_OK:
        raise ESError(rc, "plan failed")
    fs = np.zeros((nloc, nf), np.int64)
    fr = np.zeros((nloc, nf), np.int32)
    ss = np.zeros(max(ns.value, 1), np.int64)
    sc = np.zeros(world, np.int64)
    rcnt = np.zeros(world, np.int64)
    rc = es_plan(dim, ne, ev.ctypes.data_as(_lp), rank, world, fs.ctypes.data_as(_lp),
                 fr.ctypes.data_as(_ip), ss.ctypes.data_as(_lp), sc.ctypes.data_as(_lp),
                 rcnt.ctypes.data_as(_lp), ctypes.byref(ns), ctypes.byref(nh))
    if rc != ES_OK:
        raise ESError(rc, "plan failed")
    return dict(first=first, nloc=nloc, face_slot=fs, face_reflect=fr, send_slots=ss[:ns.value],
                send_count=sc, recv_count=rcnt, n_halo=nh.value)


def declared_symbols():
    """Every function name declared in include/es.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(es_[a-z_]+)\s*\(", txt)) - {"es_map_fn"})


def dp54_controller(step, T, dt0, rtol, atol, max_steps=1000000, safety=0.9, facmin=0.2, facmax=5.0):
    """Step-size control of Hairer-Norsett-Wanner I, eq. II.4.13 for an embedded pair of orders 5(4):
    dt_new = dt min(facmax, max(facmin, safety err^(-1/5))), facmax = 1 right after a rejection;
    the last step lands on T exactly.  `step(dt, rtol, atol) -> (err, accepted)` advances the state
    when accepted.  Returns (accepted, rejected, dt)."""
    t, dt, nacc, nrej, after_reject = 0.0, float(dt0), 0, 0, False
    while t < T * (1.0 - 1e-14):
        if nacc + nrej >= max_steps:
            raise ESError(-1, f"dp54: more than {max_steps} steps before T")
        h = min(dt, T - t)
        err, ok = step(h, rtol, atol)
        if not math.isfinite(err):  # a trial stage blew up (or 0/0): reject and shrink
            ok, fac = False, facmin
        else:
            fac = safety * err ** -0.2 if err > 0.0 else facmax
            fac = min(1.0 if after_reject else facmax, max(facmin, fac))
        if ok:
            t += h
            nacc += 1
            after_reject = False
        else:
            nrej += 1
            after_reject = True
        dt = h * fac
    return nacc, nrej, dt


def _group(ctxs):
    arr = (_vp * len(ctxs))(*[c.h.value if hasattr(c.h, "value") else c.h for c in ctxs])
    return arr, len(ctxs)


def _ptrs(ts):
    return (_vp * len(ts))(*[_ptr(t).value for t in ts])


def group_rhs(ctxs, us, dudts):
    """es_group_rhs: the loopback multi-rank RHS of contexts ranks 0..n-1 (one device, no NCCL)"""
    g, n = _group(ctxs)
    rc = es_group_rhs(g, n, _ptrs(us), _ptrs(dudts))
    if rc != ES_OK:
        raise ESError(rc, es_last_error(ctxs[0].h).decode())


def group_step(ctxs, dt, nsteps=1):
    g, n = _group(ctxs)
    rc = es_group_step(g, n, float(dt), int(nsteps))
    if rc != ES_OK:
        raise ESError(rc, es_last_error(ctxs[0].h).decode())


def group_entropy_production(ctxs, us):
    g, n = _group(ctxs)
    rate, sc = ctypes.c_double(), ctypes.c_double()
    cons = np.zeros(ctxs[0].d + 2)
    rc = es_group_entropy_production(g, n, _ptrs(us), ctypes.byref(rate), ctypes.byref(sc), cons.ctypes.data_as(_dp))
    if rc != ES_OK:
        raise ESError(rc, es_last_error(ctxs[0].h).decode())
    return rate.value, sc.value, cons


class ESError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"es error {code}: {msg}")
        self.code = code


def _ptr(t):
    """data pointer of a torch tensor or numpy array"""
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(t.ctypes.data)


class Context:
    """Thin owner of an es_context.  `mesh` is a dict with elem_vertices, elem_vertex_coords, period
    (e.g. es_inputs.split_cartesian); `warp` a callable [n,d] -> [n,d] (the geometry map)."""

    def __init__(self, mesh, p, warp=None, gamma=1.4, interface_flux=1, rank=0, world=1, nccl_id=None,
                 stream=None, device=0, check_admissibility=0, volume_mode=0, mapping_nodes=0,
                 metric_storage=0):
        self.d = int(mesh["d"]) if "d" in mesh else int(np.asarray(mesh["period"]).size)
        self._ev = np.ascontiguousarray(mesh["elem_vertices"], dtype=np.int64)
        self._evx = np.ascontiguousarray(mesh["elem_vertex_coords"], dtype=np.float64)
        self._per = np.ascontiguousarray(mesh["period"], dtype=np.float64)
        self.p = p
        self.ne = len(self._ev)
        d = self.d
        err = []

        def cb(user, n, xin, xout):
            try:
                xi = np.ctypeslib.as_array(xin, shape=(n * d,)).reshape(n, d)
                xo = np.ctypeslib.as_array(xout, shape=(n * d,)).reshape(n, d)
                xo[:] = warp(xi) if warp is not None else xi
            except Exception as ex:  # pragma: no cover
                err.append(ex)
        self._cb = es_map_fn(cb)
        m = es_mesh(d, self.ne, self._ev.ctypes.data_as(_lp), self._evx.ctypes.data_as(_dp),
                    self._per.ctypes.data_as(_dp))
        self._nccl_id = nccl_id
        o = es_options(gamma, interface_flux, rank, world, nccl_id, stream, device, check_admissibility, volume_mode,
                       mapping_nodes, metric_storage)
        h = _vp()
        rc = es_setup(ctypes.byref(h), ctypes.byref(m), p, self._cb, None, ctypes.byref(o))
        self.h = h
        if err:
            raise err[0]
        if rc != ES_OK:
            msg = es_last_error(h).decode() if h else ""
            raise ESError(rc, msg)
        Np, Nq, Nqf = _i(), _i(), _i()
        nloc, first = ctypes.c_int64(), ctypes.c_int64()
        es_sizes(h, ctypes.byref(Np), ctypes.byref(Nq), ctypes.byref(Nqf), ctypes.byref(nloc), ctypes.byref(first))
        self.Np, self.Nq, self.Nqf = Np.value, Nq.value, Nqf.value
        self.nloc, self.first = nloc.value, first.value
        self.Nc = d + 2
        self.shape = (self.nloc, self.Nc, self.Np)

    def _check(self, rc):
        if rc != ES_OK:
            raise ESError(rc, es_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            es_destroy(self.h)
        self.h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- device-pointer API (torch CUDA tensors) --
    def rhs(self, u, dudt):
        self._check(es_rhs(self.h, _ptr(u), _ptr(dudt)))

    def rhs_stage1(self, u):
        """entropy projection + packed boundary traces; returns the device send-buffer address"""
        b = _vp()
        self._check(es_rhs_stage1(self.h, _ptr(u), ctypes.byref(b)))
        return b.value

    def halo_buffer(self):
        b = _vp()
        self._check(es_halo_buffer(self.h, ctypes.byref(b)))
        return b.value

    def rhs_stage2(self, dudt):
        self._check(es_rhs_stage2(self.h, _ptr(dudt)))

    def rhs_host(self, u_host, dudt_host):
        self._check(es_rhs_host(self.h, _ptr(u_host), _ptr(dudt_host)))

    def set_state(self, u):
        self._check(es_set_state(self.h, _ptr(u)))

    def get_state(self, u):
        self._check(es_get_state(self.h, _ptr(u)))

    def step(self, dt, nsteps=1):
        self._check(es_step(self.h, float(dt), int(nsteps)))

    def step_dp54(self, dt, rtol=1e-6, atol=1e-8):
        """one Dormand-Prince 5(4) step (es_step_dp54): (scaled error, accepted)"""
        err, acc = ctypes.c_double(), _i()
        self._check(es_step_dp54(self.h, float(dt), float(rtol), float(atol), ctypes.byref(err), ctypes.byref(acc)))
        return err.value, bool(acc.value)

    def integrate_dp54(self, T, dt0, rtol=1e-6, atol=1e-8, max_steps=1000000):
        """adaptive Dormand-Prince 5(4) integration of the library state over [0, T] (host step-size
        control, see dp54_controller); returns (accepted steps, rejected steps, last dt)"""
        return dp54_controller(self.step_dp54, T, dt0, rtol, atol, max_steps)

    def entropy_production(self, u):
        r, a = ctypes.c_double(), ctypes.c_double()
        cons = (ctypes.c_double * 5)()
        self._check(es_entropy_production(self.h, _ptr(u), ctypes.byref(r), ctypes.byref(a),
                                          ctypes.cast(cons, _dp)))
        return r.value, a.value, np.array(cons[:self.Nc])

    def flux_counts(self):
        v, f, e = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        i = ctypes.c_double()
        self._check(es_flux_counts(self.h, ctypes.byref(v), ctypes.byref(f), ctypes.byref(e), ctypes.byref(i)))
        return dict(volume=v.value, facet=f.value, eq56=e.value, interface=i.value)

    def step_host(self, u_host_in, u_host_out, dt, nsteps=1):
        """es_step_host: host state in -> nsteps RK4 steps -> host state out (synchronous)"""
        self._check(es_step_host(self.h, _ptr(u_host_in), _ptr(u_host_out), dt, nsteps))

    def set_graphs(self, on=True):
        self._check(es_set_graphs(self.h, 1 if on else 0))

    def eval_points(self, u, xi, x_out=None, jac_out=None):
        """es_eval_points: solution at reference points xi [npts][d] (host numpy) of every local element:
        returns a device tensor [n_local][npts][N_c]; x_out / jac_out optional device tensors"""
        import torch
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        npts = xi.shape[0]
        out = torch.empty((self.nloc, npts, self.d + 2), dtype=torch.float64, device=u.device)
        self._check(es_eval_points(self.h, _ptr(u), npts, xi.ctypes.data_as(_dp), _ptr(out),
                                   _ptr(x_out) if x_out is not None else None,
                                   _ptr(jac_out) if jac_out is not None else None))
        return out

    def adv_configure(self, a, flux_mode=1, form=0):
        """linear-advection workload (es_adv_configure): velocity a [d], flux 0 central / 1 upwind,
        form 0 skew-symmetric / 1 conservative"""
        av = np.zeros(3)
        av[:len(a)] = a
        self._check(es_adv_configure(self.h, av.ctypes.data_as(_dp), int(flux_mode), int(form)))

    def adv_rhs(self, u, dudt, energy=False):
        """es_adv_rhs on device tensors [n_local][N_p]; returns (rate, scale) when energy"""
        en = np.zeros(2)
        self._check(es_adv_rhs(self.h, _ptr(u), _ptr(dudt), en.ctypes.data_as(_dp) if energy else None))
        return (en[0], en[1]) if energy else None

    def adv_step(self, u, dt, nsteps=1):
        self._check(es_adv_step(self.h, _ptr(u), float(dt), int(nsteps)))

    def step_erk(self, dt, A, b, nsteps=1):
        """es_step_erk: nsteps explicit Runge-Kutta steps with the Butcher tableau (A [s][s], b [s])"""
        A = np.ascontiguousarray(A, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        s = len(b)
        assert A.shape == (s, s)
        self._check(es_step_erk(self.h, float(dt), s, A.ctypes.data_as(_dp), b.ctypes.data_as(_dp), int(nsteps)))

    def count_fluxes(self, u):
        """flux evaluations counted in the kernels on one RHS of u (device tensor): int64 array
        [n_local][4] = volume, facet correction, issued (masked included), interface (es_count_fluxes)"""
        out = np.zeros((self.nloc, 4), np.int64)
        self._check(es_count_fluxes(self.h, _ptr(u), out.ctypes.data_as(_lp)))
        return out

    def node_coords(self, x):
        self._check(es_node_coords(self.h, _ptr(x)))

    def project_nodal(self, un, um):
        self._check(es_project_nodal(self.h, _ptr(un), _ptr(um)))

    def eval_nodal(self, um, un):
        self._check(es_eval_nodal(self.h, _ptr(um), _ptr(un)))

    def node_weights(self, wj):
        self._check(es_node_weights(self.h, _ptr(wj)))

    def element_geometry(self, k):
        d = self.d
        G = np.zeros((self.Nq, d, d))
        Jn = np.zeros((d + 1, self.Nqf, d))
        Jt = np.zeros(self.Nq)
        self._check(es_element_geometry(self.h, k, G.ctypes.data_as(_dp), Jn.ctypes.data_as(_dp),
                                        Jt.ctypes.data_as(_dp)))
        return dict(G=G, Jn=Jn, Jt=Jt)

    def synchronize(self):
        self._check(es_synchronize(self.h))

    def stream(self):
        return es_stream(self.h)

    def launch_count(self):
        return es_launch_count(self.h)

    def reset_launch_count(self):
        es_reset_launch_count(self.h)

    def timing_enable(self, on=True):
        self._check(es_timing_enable(self.h, 1 if on else 0))

    def timing_read(self, cls):
        t, n = ctypes.c_double(), ctypes.c_int64()
        self._check(es_timing_read(self.h, cls, ctypes.byref(t), ctypes.byref(n)))
        return t.value, n.value
