"""GPU <-> oracle parity of modal (compressed) metric storage (es_options.metric_storage = 1;
SURVEY 8(f) rank 4, R33) -- B200 required.

The product stores g~ = V^T W G per element (setup kernel) and expands G = V g~ in the flux kernel's
prologue (rhs2_mm_kernel); the oracle replaces G by V V^T W G (oracle/oracle.cpp
ora_mesh_use_modal_metrics, pinned in tests/test_oracle_modal_metrics.py).  Tolerance as the main
parity tests (1e-11 per conserved variable, BASELINE north_star / R20).  At sizes the oracle does not
finish, the property that holds at any size is checked: modal and nodal storage give the same RHS
and RK4 steps up to rounding (the metric terms have degree <= p).
"""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-11


@pytest.fixture(scope="module")
def es():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_07874_b200 as es
    return es


def _L(d):
    return 2.0 if d == 2 else 2.0 * math.pi


def _warp(kind, d, L, M):
    return {"paper": I.paper_warp(d, L), "bj": I.bj_warp(d, L, M), "none": None}[kind]


def _relerr(a, b):
    return np.array([np.abs(a[:, v] - b[:, v]).max() / max(np.abs(b[:, v]).max(), 1e-300) for v in range(a.shape[1])])


def _gpu_rhs(ctx, u):
    ut = torch.from_numpy(u).cuda()
    du = torch.empty_like(ut)
    ctx.rhs(ut, du)
    ctx.synchronize()
    return du.cpu().numpy()


CASES = [
    # d, M, p, warp, flux mode
    (2, 3, 2, "paper", 1),
    (2, 4, 4, "bj", 1),
    (2, 3, 5, "paper", 0),
    (2, 3, 10, "paper", 1),   # C3 degree
    (3, 3, 1, "paper", 1),
    (3, 3, 2, "paper", 1),
    (3, 3, 3, "paper", 1),    # even line length
    (3, 3, 4, "bj", 0),       # C4 family, EC
    (3, 3, 6, "paper", 1),
    (3, 3, 8, "paper", 1),    # C5 degree on the hardest geometry
    (3, 3, 8, "bj", 2),
]


@pytest.mark.parametrize("d,M,p,warp,fm", CASES)
def test_modal_metric_rhs_parity(es, d, M, p, warp, fm):
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = _warp(warp, d, L, M)
    om = O.Mesh(mesh, p, warp=w, metric_storage=1)
    x = om.node_coords()
    u = om.project(I.density_wave(x, L) if d == 2 else I.taylor_green(x, Ma=0.3))
    u = I.perturb_modal(u, d, p, seed=2, amp=1e-2)
    ref, _ = om.rhs(u, flux_mode=fm, variant=1)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm, metric_storage=1)
    got = _gpu_rhs(ctx, u)
    err = _relerr(got, ref)
    assert err.max() < TOL, err


@pytest.mark.parametrize("d,M,p", [(2, 16, 4), (3, 8, 8)])
def test_modal_metric_equals_nodal_at_size(es, d, M, p):
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = I.bj_warp(d, L, M)
    u = I.modal_state_from_centroids(mesh, p, "tgv" if d == 3 else "density_wave", seed=5, amp=1e-2)
    cn = es.Context(mesh, p, warp=w, interface_flux=1)
    cm = es.Context(mesh, p, warp=w, interface_flux=1, metric_storage=1)
    dn, dm = _gpu_rhs(cn, u), _gpu_rhs(cm, u)
    assert _relerr(dm, dn).max() < 1e-12
    # RK4 steps through the CUDA-graph path
    dt = 1e-4
    outs = []
    for c in (cn, cm):
        c.set_state(torch.from_numpy(u).cuda())
        c.step(dt, 3)
        o = torch.empty((c.nloc, d + 2, c.Np), dtype=torch.float64, device="cuda")
        c.get_state(o)
        c.synchronize()
        outs.append(o.cpu().numpy())
    assert np.abs(outs[1] - outs[0]).max() < 1e-13 * np.abs(outs[0]).max()


def test_metric_storage_option_checked(es):
    mesh = I.split_cartesian(2, 3, 2.0)
    with pytest.raises(es.ESError):
        es.Context(mesh, 2, metric_storage=2)
