"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module.  The product path (paper_2312_07874_b200/) never imports it and shares no code with it.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_int64)
MAPFN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_int64, _dp, _dp)


class Stats(ctypes.Structure):
    _fields_ = [("volume_pairs", ctypes.c_int64), ("facet_pairs", ctypes.c_int64),
                ("interface_evals", ctypes.c_int64), ("series_branch", ctypes.c_int64),
                ("log_branch", ctypes.c_int64), ("n_elements", ctypes.c_int64),
                ("entropy_rate", ctypes.c_double), ("entropy_abs", ctypes.c_double),
                ("conservation", ctypes.c_double * 5), ("inadmissible", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            from tools.build import build_oracle
            build_oracle()
        L = ctypes.CDLL(LIB_PATH)
        L.ora_jacobi.restype = ctypes.c_double
        L.ora_jacobi.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double]
        L.ora_jacobi_deriv.restype = ctypes.c_double
        L.ora_jacobi_deriv.argtypes = L.ora_jacobi.argtypes
        L.ora_gauss_jacobi.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp, _dp]
        L.ora_lagrange_diff.argtypes = [ctypes.c_int, _dp, _dp]
        L.ora_ref_sizes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip]
        L.ora_ref_get.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p, _dp]
        L.ora_pkd_eval.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp]
        for nm in ("ora_entropy_vars", "ora_cons_from_entropy"):
            getattr(L, nm).argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, _dp]
        L.ora_euler_flux.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp]
        L.ora_ec_flux.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp, _dp]
        L.ora_es_flux.argtypes = L.ora_ec_flux.argtypes
        L.ora_ej_flux.argtypes = L.ora_ec_flux.argtypes
        L.ora_md_flux.argtypes = L.ora_ec_flux.argtypes
        L.ora_dudw.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, _dp]
        L.ora_wave_speed.restype = ctypes.c_double
        L.ora_wave_speed.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _dp, _dp]
        L.ora_ln_mean.restype = ctypes.c_double
        L.ora_ln_mean.argtypes = [ctypes.c_double, ctypes.c_double]
        L.ora_inv_ln_mean.restype = ctypes.c_double
        L.ora_inv_ln_mean.argtypes = [ctypes.c_double, ctypes.c_double]
        L.ora_entropy.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, _dp, _dp, _dp]
        L.ora_mesh_create.restype = ctypes.c_void_p
        L.ora_mesh_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, _lp, _dp, _dp, MAPFN,
                                      ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, _lp]
        L.ora_mesh_create2.restype = ctypes.c_void_p
        L.ora_mesh_create2.argtypes = L.ora_mesh_create.argtypes + [ctypes.c_int]
        L.ora_nodes.restype = ctypes.c_int
        L.ora_nodes.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.ora_mesh_destroy.argtypes = [ctypes.c_void_p]
        L.ora_mesh_geometry.argtypes = [ctypes.c_void_p, ctypes.c_int64, _dp, _dp, _dp, _dp, _dp]
        L.ora_mesh_conn.argtypes = [ctypes.c_void_p, _lp, _ip, _ip]
        L.ora_metric_modal.argtypes = [ctypes.c_void_p, ctypes.c_int64, _dp]
        L.ora_mesh_use_modal_metrics.argtypes = [ctypes.c_void_p]
        L.ora_project.argtypes = [ctypes.c_void_p, ctypes.c_int64, _lp, _dp, _dp]
        L.ora_rhs.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _lp,
                              ctypes.c_int, ctypes.POINTER(Stats)]
        L.ora_rk4.argtypes = [ctypes.c_void_p, _dp, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.ora_dp54_tableau.argtypes = [_dp, _dp, _dp, _dp]
        L.ora_advection_rhs.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int, ctypes.c_int, _dp, _dp]
        L.ora_dp54.argtypes = [ctypes.c_void_p, _dp, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
                               ctypes.c_int, _dp, _dp]
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(_dp)


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def gauss_jacobi(q, a, b):
    x = np.zeros(q + 1)
    w = np.zeros(q + 1)
    lib().ora_gauss_jacobi(q, a, b, _d(x), _d(w))
    return x, w


def jacobi(n, a, b, x):
    return lib().ora_jacobi(n, a, b, x)


def jacobi_deriv(n, a, b, x):
    return lib().ora_jacobi_deriv(n, a, b, x)


def lagrange_diff(nodes):
    nodes = _c(nodes)
    n = len(nodes)
    D = np.zeros((n, n))
    lib().ora_lagrange_diff(n, _d(nodes), _d(D))
    return D


def ref_sizes(d, q, p=None):
    out = (ctypes.c_int * 5)()
    lib().ora_ref_sizes(d, q, q if p is None else p, out)
    return dict(n=out[0], Nq=out[1], Nf=out[2], Nqf=out[3], Np=out[4])


_SHAPES = {
    "eta1": lambda d, s: (s["n"],), "w1": lambda d, s: (s["n"],), "eta3": lambda d, s: (s["n"],),
    "w3": lambda d, s: (s["n"],), "xi": lambda d, s: (s["Nq"], d), "eta": lambda d, s: (s["Nq"], d),
    "W": lambda d, s: (s["Nq"],), "xif": lambda d, s: (s["Nf"], s["Nqf"], d),
    "B": lambda d, s: (s["Nf"], s["Nqf"]), "nhat": lambda d, s: (s["Nf"], d),
    "D": lambda d, s: (d, s["Nq"], s["Nq"]), "Q": lambda d, s: (d, s["Nq"], s["Nq"]),
    "E": lambda d, s: (d, s["Nq"], s["Nq"]), "S": lambda d, s: (d, s["Nq"], s["Nq"]),
    "R": lambda d, s: (s["Nf"], s["Nqf"], s["Nq"]), "V": lambda d, s: (s["Nq"], s["Np"]),
    "alpha": lambda d, s: (s["Np"], d),
}


def ref_get(d, q, name, p=None):
    p = q if p is None else p
    s = ref_sizes(d, q, p)
    out = np.zeros(_SHAPES[name](d, s))
    rc = lib().ora_ref_get(d, q, p, name.encode(), _d(out))
    assert rc == 0
    return out


def pkd_eval(d, p, xi):
    xi = _c(np.atleast_2d(xi))
    Np = ref_sizes(d, p, p)["Np"]
    vals = np.zeros((len(xi), Np))
    grads = np.zeros((len(xi), Np, d))
    lib().ora_pkd_eval(d, p, len(xi), _d(xi), _d(vals), _d(grads))
    return vals, grads


def entropy_vars(U, gamma=1.4):
    U = _c(np.atleast_2d(U))
    W = np.zeros_like(U)
    lib().ora_entropy_vars(U.shape[1] - 2, gamma, len(U), _d(U), _d(W))
    return W


def cons_from_entropy(W, gamma=1.4):
    W = _c(np.atleast_2d(W))
    U = np.zeros_like(W)
    lib().ora_cons_from_entropy(W.shape[1] - 2, gamma, len(W), _d(W), _d(U))
    return U


def euler_flux(U, nvec, gamma=1.4):
    U = _c(np.atleast_2d(U))
    nvec = _c(np.broadcast_to(nvec, (len(U), U.shape[1] - 2)))
    F = np.zeros_like(U)
    lib().ora_euler_flux(U.shape[1] - 2, gamma, len(U), _d(U), _d(nvec), _d(F))
    return F


def ec_flux(Ua, Ub, nvec, gamma=1.4):
    Ua = _c(np.atleast_2d(Ua))
    Ub = _c(np.atleast_2d(Ub))
    nvec = _c(np.broadcast_to(nvec, (len(Ua), Ua.shape[1] - 2)))
    F = np.zeros_like(Ua)
    lib().ora_ec_flux(Ua.shape[1] - 2, gamma, len(Ua), _d(Ua), _d(Ub), _d(nvec), _d(F))
    return F


def es_flux(Ua, Ub, nunit, gamma=1.4):
    Ua = _c(np.atleast_2d(Ua))
    Ub = _c(np.atleast_2d(Ub))
    nunit = _c(np.broadcast_to(nunit, (len(Ua), Ua.shape[1] - 2)))
    F = np.zeros_like(Ua)
    lib().ora_es_flux(Ua.shape[1] - 2, gamma, len(Ua), _d(Ua), _d(Ub), _d(nunit), _d(F))
    return F


def ej_flux(Ua, Ub, nunit, gamma=1.4):
    """entropy-jump scalar dissipation interface flux (flux_mode 2, reading R27)"""
    Ua = _c(np.atleast_2d(Ua))
    Ub = _c(np.atleast_2d(Ub))
    nunit = _c(np.broadcast_to(nunit, (len(Ua), Ua.shape[1] - 2)))
    F = np.zeros_like(Ua)
    lib().ora_ej_flux(Ua.shape[1] - 2, gamma, len(Ua), _d(Ua), _d(Ub), _d(nunit), _d(F))
    return F


def md_flux(Ua, Ub, nunit, gamma=1.4):
    """matrix-dissipation interface flux (flux_mode 3, reading R28)"""
    Ua = _c(np.atleast_2d(Ua))
    Ub = _c(np.atleast_2d(Ub))
    nunit = _c(np.broadcast_to(nunit, (len(Ua), Ua.shape[1] - 2)))
    F = np.zeros_like(Ua)
    lib().ora_md_flux(Ua.shape[1] - 2, gamma, len(Ua), _d(Ua), _d(Ub), _d(nunit), _d(F))
    return F


def dudw(U, gamma=1.4):
    """du/dw at each state [n][d+2][d+2] (reading R27)"""
    U = _c(np.atleast_2d(U))
    n = U.shape[1]
    A = np.zeros((len(U), n, n))
    lib().ora_dudw(n - 2, gamma, len(U), _d(U), _d(A))
    return A


def wave_speed(Ua, Ub, nunit, gamma=1.4):
    Ua, Ub, nunit = _c(Ua), _c(Ub), _c(nunit)
    return lib().ora_wave_speed(len(Ua) - 2, gamma, _d(Ua), _d(Ub), _d(nunit))


def dp54_tableau():
    c, a, b, bh = np.zeros(7), np.zeros((7, 7)), np.zeros(7), np.zeros(7)
    lib().ora_dp54_tableau(_d(c), _d(a), _d(b), _d(bh))
    return c, a, b, bh


def ln_mean(x, y):
    return lib().ora_ln_mean(x, y)


def inv_ln_mean(x, y):
    return lib().ora_inv_ln_mean(x, y)


def entropy(U, gamma=1.4):
    U = _c(np.atleast_2d(U))
    d = U.shape[1] - 2
    S = np.zeros(len(U))
    F = np.zeros((len(U), d))
    lib().ora_entropy(d, gamma, len(U), _d(U), _d(S), _d(F))
    return S, F


class Mesh:
    """Oracle mesh + geometry.  `mesh` is an es_inputs.split_cartesian dict, `warp` a callable
    [n,d] -> [n,d] (the user map).  `active`: optional element subset (plus neighbours)."""

    def __init__(self, mesh, p, warp=None, gamma=1.4, active=None, nodes=0, metric_storage=0):
        self.d = mesh["d"]
        self.p = p
        self.gamma = gamma
        self.ne = len(mesh["elem_vertices"])
        s = ref_sizes(self.d, p, p)
        self.Nq, self.Nf, self.Nqf, self.Np, self.n = s["Nq"], s["Nf"], s["Nqf"], s["Np"], s["n"]
        self.Nc = self.d + 2
        ev = _c(mesh["elem_vertices"], np.int64)
        evx = _c(mesh["elem_vertex_coords"])
        per = _c(mesh["period"])
        d = self.d
        err = []

        def cb(user, n, xin, xout):
            try:
                xi = np.ctypeslib.as_array(xin, shape=(n * d,)).reshape(n, d)
                xo = np.ctypeslib.as_array(xout, shape=(n * d,)).reshape(n, d)
                xo[:] = warp(xi) if warp is not None else xi
            except Exception as ex:  # pragma: no cover
                err.append(ex)
        self._cb = MAPFN(cb)
        if active is None:
            act_p, nact = None, 0
        else:
            self._act = _c(active, np.int64)
            act_p, nact = self._act.ctypes.data_as(_lp), len(self._act)
        h = lib().ora_mesh_create2(d, p, self.ne, ev.ctypes.data_as(_lp), _d(evx), _d(per), self._cb, None,
                                   gamma, nact, act_p, int(nodes))
        if err:
            raise err[0]
        if not h:
            raise RuntimeError("oracle mesh creation failed")
        self.h = h
        if metric_storage:  # modal metric storage: G -> V V^T W G
            lib().ora_mesh_use_modal_metrics(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ora_mesh_destroy(self.h)
            self.h = None

    def geometry(self, e):
        d, Nq, Nf, Nqf = self.d, self.Nq, self.Nf, self.Nqf
        G = np.zeros((Nq, d, d))
        Gf = np.zeros((Nf, Nqf, d, d))
        Jt = np.zeros(Nq)
        Jn = np.zeros((Nf, Nqf, d))
        xq = np.zeros((Nq, d))
        rc = lib().ora_mesh_geometry(self.h, e, _d(G), _d(Gf), _d(Jt), _d(Jn), _d(xq))
        if rc:
            raise KeyError(e)
        return dict(G=G, Gf=Gf, Jt=Jt, Jn=Jn, xq=xq)

    def metric_modal(self, e):
        """PKD coefficients of the volume metric of element e: [d*d][Np], row l*d + m = V^T W G_lm"""
        gm = np.zeros((self.d * self.d, self.Np))
        if lib().ora_metric_modal(self.h, e, _d(gm)):
            raise KeyError(e)
        return gm

    def conn(self):
        nbr = np.zeros((self.ne, self.Nf), np.int64)
        nf = np.zeros((self.ne, self.Nf), np.int32)
        rf = np.zeros((self.ne, self.Nf), np.int32)
        lib().ora_mesh_conn(self.h, nbr.ctypes.data_as(_lp), nf.ctypes.data_as(_ip), rf.ctypes.data_as(_ip))
        return nbr, nf, rf

    def node_coords(self, elems=None):
        elems = range(self.ne) if elems is None else elems
        return np.stack([self.geometry(e)["xq"] for e in elems])

    def project(self, u_nodal, elems=None):
        """u_nodal [ne or len(elems)][Nq][Nc] -> modal [ne][Nc][Np] (rows of elems)."""
        if elems is None:
            elems = np.arange(self.ne)
            full = _c(u_nodal)
        else:
            elems = np.asarray(elems, np.int64)
            full = np.zeros((self.ne, self.Nq, self.Nc))
            full[elems] = u_nodal
        el = _c(elems, np.int64)
        out = np.zeros((self.ne, self.Nc, self.Np))
        lib().ora_project(self.h, len(el), el.ctypes.data_as(_lp), _d(full), _d(out))
        return out

    def rhs(self, u, flux_mode=1, variant=1, elems=None, nthreads=0):
        u = _c(u)
        out = np.zeros_like(u)
        st = Stats()
        if elems is None:
            rc = lib().ora_rhs(self.h, _d(u), _d(out), flux_mode, variant, 0, None, nthreads, ctypes.byref(st))
        else:
            el = _c(elems, np.int64)
            rc = lib().ora_rhs(self.h, _d(u), _d(out), flux_mode, variant, len(el), el.ctypes.data_as(_lp),
                               nthreads, ctypes.byref(st))
        if rc == 3:
            raise FloatingPointError("inadmissible state")
        if rc:
            raise RuntimeError(f"ora_rhs failed ({rc})")
        return out, st

    def dp54(self, u, dt, rtol=1e-6, atol=1e-8, flux_mode=1, nthreads=0):
        """one Dormand-Prince 5(4) step: (u5, scaled RMS error estimate)"""
        u = np.ascontiguousarray(u, dtype=np.float64)
        u5 = np.zeros_like(u)
        err = ctypes.c_double()
        rc = lib().ora_dp54(self.h, _d(u), dt, rtol, atol, flux_mode, nthreads, _d(u5), ctypes.byref(err))
        if rc:
            raise RuntimeError(f"ora_dp54 failed ({rc})")
        return u5, err.value

    def advection_rhs(self, u, a, flux_mode=1, form=0):
        """linear advection: u [ne][Np] (or [ne][1][Np]) modal scalar, velocity a [d];
        form 0 skew-symmetric [eq:rhs_skew], 1 conservative; flux_mode 0 central, 1 upwind.
        Returns (dudt [ne][Np], energy rate sum u^T r, energy scale sum |u_i r_i|)."""
        u = _c(np.asarray(u).reshape(self.ne, -1))
        av = _c(np.asarray(a, dtype=np.float64).reshape(-1))
        out = np.zeros_like(u)
        en = np.zeros(2)
        rc = lib().ora_advection_rhs(self.h, _d(u), _d(av), flux_mode, form, _d(out), _d(en))
        if rc:
            raise RuntimeError(f"ora_advection_rhs failed ({rc})")
        return out, en[0], en[1]

    def advection_rk4(self, u, a, dt, nsteps, flux_mode=1, form=0):
        """classical RK4 (R17) on the advection right-hand side (Python loop over the oracle's RHS)"""
        u = np.array(np.asarray(u).reshape(self.ne, -1), dtype=np.float64)
        for _ in range(nsteps):
            k1 = self.advection_rhs(u, a, flux_mode, form)[0]
            k2 = self.advection_rhs(u + 0.5 * dt * k1, a, flux_mode, form)[0]
            k3 = self.advection_rhs(u + 0.5 * dt * k2, a, flux_mode, form)[0]
            k4 = self.advection_rhs(u + dt * k3, a, flux_mode, form)[0]
            u = u + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
        return u

    def rk4(self, u, dt, nsteps, flux_mode=1, nthreads=0):
        u = np.array(u, dtype=np.float64, copy=True, order="C")
        rc = lib().ora_rk4(self.h, _d(u), dt, nsteps, flux_mode, nthreads)
        if rc:
            raise RuntimeError(f"ora_rk4 failed ({rc})")
        return u


def nodes(d, N, family):
    """Mapping / curl-interpolation node set of degree N on the reference simplex: family 0 = the
    equispaced lattice (R10), 1 = warp & blend (R32).  Returns (xi [M, d], lam [M, d+1])."""
    M = math.comb(N + d, d)
    xi = np.zeros((M, d))
    lam = np.zeros((M, d + 1))
    m = lib().ora_nodes(d, N, family, _d(xi), _d(lam))
    assert m == M
    return xi, lam
