"""Pins of the oracle's linear-advection workload: the skew-symmetric weak form
P:431-436 [eq:rhs_skew] against what the paper and the mathematics fix:
  * energy conservation with a central flux on CURVED periodic meshes ("to ensure energy
    stability for linear problems on curvilinear meshes, a property which cannot be guaranteed for
    discretizations in the form of [eq:rhs_cons]") -- and the conservative form does not conserve it;
  * energy dissipation with the upwind flux;
  * on affine meshes the two forms coincide (the difference 1/2 (Q + Q^T) G f = 1/2 E G f cancels the
    surface term's 1/2 N R f by the SBP property);
  * free-stream (constant) preservation on curved meshes (the discrete metric identities);
  * order p + 1 for a translating sine wave with the upwind flux (the exact solution is the initial
    data shifted by a t).
"""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O


def _setup(d, M, p, warp):
    L = 2.0 if d == 2 else 2.0 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = I.paper_warp(d, L) if warp else None
    om = O.Mesh(mesh, p, warp=w)
    return L, om


def _wave(om, L, d, t=0.0, a=None):
    x = om.node_coords()
    a = np.zeros(d) if a is None else np.asarray(a)
    u0 = 1.0 + 0.3 * np.sin(2 * math.pi / L * (x - a * t).sum(-1))
    return om.project(np.repeat(u0[..., None], d + 2, -1))[:, 0, :]


A = {2: [1.0, -0.5], 3: [1.0, -0.5, 0.3]}


@pytest.mark.parametrize("d,p", [(2, 2), (2, 4), (3, 2), (3, 3)])
def test_skew_form_conserves_energy_on_curved_meshes(d, p):
    L, om = _setup(d, 3, p, True)
    u = I.perturb_modal(_wave(om, L, d)[:, None, :], d, p, seed=1, amp=1e-2)[:, 0, :]
    _, er, ea = om.advection_rhs(u, A[d], flux_mode=0, form=0)
    assert abs(er) <= 1e-13 * ea, (er, ea)
    _, er_c, ea_c = om.advection_rhs(u, A[d], flux_mode=0, form=1)
    if (d, p) != (2, 2):  # 2D p = 2: J~ = J and the forms coincide (R13 note), otherwise they differ
        assert abs(er_c) > 1e-6 * ea_c  # the conservative form does not conserve energy on curved meshes
    _, er_u, ea_u = om.advection_rhs(u, A[d], flux_mode=1, form=0)
    assert er_u < -1e-6 * ea_u  # upwind dissipates


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2)])
def test_affine_skew_equals_conservative_and_free_stream(d, p):
    L, om = _setup(d, 3, p, False)
    u = _wave(om, L, d)
    r0 = om.advection_rhs(u, A[d], 1, 0)[0]
    r1 = om.advection_rhs(u, A[d], 1, 1)[0]
    assert np.abs(r0 - r1).max() <= 1e-12 * np.abs(r1).max()
    L, om = _setup(d, 3, p, True)
    c = om.project(np.ones(om.node_coords().shape[:-1] + (d + 2,)))[:, 0, :]
    assert np.abs(om.advection_rhs(c, A[d], 1, 0)[0]).max() < 1e-12


def test_upwind_sine_wave_converges_at_order_p_plus_1():
    d, p, T = 2, 3, 0.5
    errs = []
    for M in (8, 16):
        L, om = _setup(d, M, p, True)
        u = _wave(om, L, d)
        h = L / M
        nst = int(math.ceil(T / (0.1 * h / ((2 * p + 1) * 1.2))))
        u = om.advection_rk4(u, A[d], T / nst, nst, flux_mode=1, form=0)
        ex = _wave(om, L, d, T, A[d])
        V = O.ref_get(d, p, "V")
        W = O.ref_get(d, p, "W")
        err = math.sqrt(sum(np.sum(W * om.geometry(e)["Jt"] * (V @ (u[e] - ex[e])) ** 2) for e in range(om.ne)))
        errs.append(err)
    order = math.log2(errs[0] / errs[1])
    assert abs(order - (p + 1)) <= 0.3, (errs, order)  # measured 4.08 (M = 8 -> 16)
