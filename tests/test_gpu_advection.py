"""GPU <-> oracle parity of the linear-advection workload: the skew-
symmetric weak form (energy stable on curved meshes) and the conservative form, central and upwind
fluxes, weight-adjusted inverse, RK4.  Tolerance as for the Euler RHS (R20): max |du_gpu - du_ora| /
max |du_ora| <= 1e-11."""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

A = {2: [1.0, -0.5], 3: [1.0, -0.5, 0.3]}


@pytest.fixture(scope="module")
def es():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_07874_b200 as es
    return es


def _setup(es, d, M, p, warp=True):
    L = 2.0 if d == 2 else 2.0 * math.pi
    mesh = I.split_cartesian(d, M, L)
    w = I.paper_warp(d, L) if warp else None
    om = O.Mesh(mesh, p, warp=w)
    x = om.node_coords()
    u0 = 1.0 + 0.3 * np.sin(2 * math.pi / L * x.sum(-1))
    u = om.project(np.repeat(u0[..., None], d + 2, -1))
    u = I.perturb_modal(u, d, p, seed=4, amp=1e-2)[:, 0, :].copy()
    ctx = es.Context(mesh, p, warp=w)
    return om, ctx, u


@pytest.mark.parametrize("d,p,fm,form", [(2, 2, 1, 0), (2, 3, 0, 0), (2, 4, 1, 1), (2, 7, 1, 0), (3, 2, 1, 0),
                                         (3, 3, 0, 0), (3, 3, 1, 1), (3, 5, 1, 0)])
def test_advection_rhs_parity(es, d, p, fm, form):
    om, ctx, u = _setup(es, d, 3, p)
    ref, er, ea = om.advection_rhs(u, A[d], flux_mode=fm, form=form)
    ctx.adv_configure(A[d], fm, form)
    ut = torch.from_numpy(u).cuda()
    du = torch.empty_like(ut)
    rate, scale = ctx.adv_rhs(ut, du, energy=True)
    got = du.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()
    assert abs(rate - er) <= 1e-12 * ea and abs(scale - ea) <= 1e-12 * ea
    if form == 0 and fm == 0:  # energy conserved to roundoff by the skew form
        assert abs(rate) <= 1e-13 * scale
    if fm == 1:
        assert rate < 0


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2)])
def test_advection_rk4_parity(es, d, p):
    om, ctx, u = _setup(es, d, 3, p)
    dt = 2e-3
    ref = om.advection_rk4(u, A[d], dt, 5, flux_mode=1, form=0)
    ctx.adv_configure(A[d], 1, 0)
    ut = torch.from_numpy(u).cuda()
    ctx.adv_step(ut, dt, 5)
    ctx.synchronize()
    got = ut.cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs((got - u) - (ref - u)).max() <= 1e-10 * np.abs(ref - u).max()
