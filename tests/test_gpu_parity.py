"""GPU <-> oracle parity of the sm_100a ES modal DSEM right-hand side (B200 required).

Tolerance (BASELINE.json north_star, reading R20): per conserved variable e,
    max_{k,i} |du_gpu - du_ora| / max_{k,i} |du_ora| <= 1e-11,
free-stream states use an absolute bound relative to the flux scale.  Integer flux counts must match
exactly.  Inputs are seeded and identical for both sides: modal coefficients are produced by the
oracle's projection of the analytic initial data (small meshes) or by es_inputs directly (full-size
meshes), never by the CUDA path.
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


def _ic(kind, x, d, L):
    if kind == "tgv":
        return I.taylor_green(x, Ma=0.1)
    if kind == "tgv3":
        return I.taylor_green(x, Ma=0.3)
    if kind == "wave":
        return I.density_wave(x, L)
    if kind == "vortex":
        return I.isentropic_vortex(x, L)
    return I.free_stream(x, d)


def _setup(es, d, M, p, warp, ic, fm, seed=1):
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = _warp(warp, d, L, M)
    om = O.Mesh(mesh, p, warp=w)
    u = om.project(_ic(ic, om.node_coords(), d, L))
    u = I.perturb_modal(u, d, p, seed=seed, amp=1e-2)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm)
    return mesh, om, ctx, u


def _relerr(a, b):
    d = a.shape[1]
    out = []
    for v in range(d):
        out.append(np.abs(a[:, v] - b[:, v]).max() / max(np.abs(b[:, v]).max(), 1e-300))
    return np.array(out)


def _gpu_rhs(ctx, u):
    ut = torch.from_numpy(u).cuda()
    du = torch.empty_like(ut)
    ctx.rhs(ut, du)
    ctx.synchronize()
    return du.cpu().numpy()


CASES = [
    # d, M, p, warp, ic, flux mode
    (2, 4, 2, "none", "vortex", 1),    # C1 geometry (affine), p = 2
    (2, 3, 3, "paper", "wave", 1),     # even line length
    (2, 4, 4, "bj", "wave", 1),        # C2 family
    (2, 3, 4, "paper", "vortex", 0),   # EC
    (2, 3, 6, "paper", "wave", 1),
    (2, 3, 10, "bj", "vortex", 1),     # C3 degree
    (3, 3, 2, "paper", "tgv3", 1),
    (3, 3, 3, "paper", "tgv3", 1),     # even line length
    (3, 3, 4, "bj", "tgv", 0),         # C4 family, EC
    (3, 3, 4, "paper", "tgv3", 1),
    (3, 3, 6, "paper", "tgv3", 1),
    (3, 3, 8, "bj", "tgv", 1),         # C5 degree
    (3, 3, 5, "paper", "tgv3", 1),     # even line length, 3D
    (3, 3, 7, "paper", "tgv3", 0),     # even line length, 3D, EC
    (3, 3, 1, "paper", "tgv3", 1),     # p = 1: two nodes per line
    (2, 3, 1, "paper", "wave", 1),
    (2, 3, 8, "paper", "wave", 1),
    (2, 3, 9, "bj", "vortex", 0),
    (3, 4, 8, "paper", "tgv3", 0),     # C5 degree on the hardest geometry, EC
    (2, 3, 4, "paper", "wave", 2),     # entropy-jump dissipation (R27)
    (3, 3, 3, "paper", "tgv3", 2),
    (3, 3, 8, "bj", "tgv", 2),
    (2, 3, 4, "paper", "vortex", 3),   # matrix dissipation (R28)
    (3, 3, 3, "paper", "tgv3", 3),
    (3, 3, 8, "bj", "tgv", 3),
]


@pytest.mark.parametrize("d,M,p,warp,ic,fm", CASES)
def test_rhs_parity(es, d, M, p, warp, ic, fm):
    mesh, om, ctx, u = _setup(es, d, M, p, warp, ic, fm)
    got = _gpu_rhs(ctx, u)
    # against the paper's own Eq. 56 nonzero iteration (oracle variant 0) -- the
    # reference that shares no pairing structure with the kernel -- and against the line-wise
    # variant 1 (one flux per unordered line pair)
    ref0, st0 = om.rhs(u, flux_mode=fm, variant=0)
    err0 = _relerr(got, ref0)
    assert (err0 <= TOL).all(), err0
    ref, st = om.rhs(u, flux_mode=fm, variant=1)
    err = _relerr(got, ref)
    assert (err <= TOL).all(), err
    _check_counts(ctx, om, u, st, st0)


def _check_counts(ctx, om, u, st, st0=None):
    # flux evaluations COUNTED IN THE KERNELS (es_count_fluxes), per element, against the pairs the
    # oracle's loops counted (R22): exact integers, identical for every element
    cnt = ctx.count_fluxes(torch.from_numpy(u).cuda())
    ne = om.ne
    assert (cnt[:, 0] == cnt[0, 0]).all() and (cnt[:, 1] == cnt[0, 1]).all()
    assert cnt[:, 0].sum() == st.volume_pairs, (cnt[0], st.volume_pairs / ne)
    assert cnt[:, 1].sum() == st.facet_pairs, (cnt[0], st.facet_pairs / ne)
    assert cnt[:, 3].sum() == st.interface_evals, (cnt[0], st.interface_evals / ne)
    assert (cnt[:, 2] >= cnt[:, 0] + cnt[:, 1]).all()  # issued includes masked jobs
    # the closed forms the library reports agree with what the kernel did
    c = ctx.flux_counts()
    assert c["volume"] == cnt[0, 0] and c["facet"] == cnt[0, 1]
    if st0 is not None:  # the paper's Eq. num_fluxes count from the oracle's variant 0
        assert c["eq56"] * ne == st0.volume_pairs + st0.facet_pairs


def test_free_stream_gpu(es):
    for d, p in ((2, 4), (3, 3)):
        L = _L(d)
        mesh = I.split_cartesian(d, 3, L)
        w = I.paper_warp(d, L)
        om = O.Mesh(mesh, p, warp=w)
        u = om.project(I.free_stream(om.node_coords(), d))
        ctx = es.Context(mesh, p, warp=w, interface_flux=1)
        got = _gpu_rhs(ctx, u)
        assert np.abs(got).max() < 1e-10


@pytest.mark.parametrize("d,p", [(2, 3), (3, 3)])
def test_geometry_and_nodes_parity(es, d, p):
    L = _L(d)
    mesh = I.split_cartesian(d, 3, L)
    w = I.paper_warp(d, L)
    om = O.Mesh(mesh, p, warp=w)
    ctx = es.Context(mesh, p, warp=w)
    x = torch.empty((ctx.nloc, ctx.Nq, d), dtype=torch.float64, device="cuda")
    ctx.node_coords(x)
    xg = x.cpu().numpy()
    for e in (0, 7, om.ne - 1):
        go = om.geometry(e)
        gg = ctx.element_geometry(e)
        assert np.abs(gg["G"] - go["G"]).max() < 1e-12 * np.abs(go["G"]).max()
        assert np.abs(gg["Jn"] - go["Jn"]).max() < 1e-12 * np.abs(go["Jn"]).max()
        assert np.abs(gg["Jt"] - go["Jt"]).max() < 1e-12 * np.abs(go["Jt"]).max()
        assert np.abs(xg[e] - go["xq"]).max() < 1e-12 * L
    # projection of nodal data (R18)
    un = I.density_wave(xg, L) if d == 2 else I.taylor_green(xg, 0.3)
    um = torch.empty((ctx.nloc, d + 2, ctx.Np), dtype=torch.float64, device="cuda")
    ctx.project_nodal(torch.from_numpy(np.ascontiguousarray(un)).cuda(), um)
    ref = om.project(un)
    assert np.abs(um.cpu().numpy() - ref).max() < 1e-12 * np.abs(ref).max()


@pytest.mark.parametrize("d,p,fm", [(2, 3, 1), (3, 2, 0), (3, 3, 1), (2, 3, 2), (3, 3, 2), (2, 3, 3), (3, 3, 3)])
def test_entropy_production_parity(es, d, p, fm):
    mesh, om, ctx, u = _setup(es, d, 3, p, "paper", "wave" if d == 2 else "tgv3", fm)
    ref, st = om.rhs(u, flux_mode=fm, variant=1)
    rate, scale, cons = ctx.entropy_production(torch.from_numpy(u).cuda())
    if fm == 0:
        assert abs(rate) < 1e-12 * st.entropy_abs
    else:
        assert rate < 0 and abs(rate - st.entropy_rate) < 1e-10 * st.entropy_abs
    assert np.abs(cons).max() < 1e-12 * om.ne * np.abs(ref).max()


@pytest.mark.parametrize("d,p", [(2, 2), (3, 2)])
def test_rk4_steps_parity(es, d, p):
    # C1-style: 10 RK4 steps on the library state vs the oracle's RK4 (R17)
    mesh, om, ctx, u = _setup(es, d, 4 if d == 2 else 3, p, "none" if d == 2 else "paper",
                              "vortex" if d == 2 else "tgv3", 1)
    dt = 1e-3
    ref = om.rk4(u, dt, 10, flux_mode=1)
    ut = torch.from_numpy(u).cuda()
    ctx.set_state(ut)
    ctx.step(dt, 10)
    out = torch.empty_like(ut)
    ctx.get_state(out)
    ctx.synchronize()
    got = out.cpu().numpy()
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-13, err
    # the update itself: compare the increments
    inc = _relerr(got - u, ref - u)
    assert (inc < 1e-10).all(), inc


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2)])
def test_dp54_step_parity(es, d, p):
    # es_step_dp54 against the oracle's Dormand-Prince 5(4) step: the 5th-order solution, the scaled
    # error estimate, rejection leaving the state unchanged, and first-same-as-last over two steps
    mesh, om, ctx, u = _setup(es, d, 3, p, "paper", "wave" if d == 2 else "tgv3", 1)
    dt, rtol, atol = 2e-3, 1e-4, 1e-6
    u1, e1 = om.dp54(u, dt, rtol, atol, flux_mode=1)
    u2, e2 = om.dp54(u1, dt, rtol, atol, flux_mode=1)
    ut = torch.from_numpy(u).cuda()
    ctx.set_state(ut)
    out = torch.empty_like(ut)
    # a tolerance far below reach: rejected, state unchanged
    err, ok = ctx.step_dp54(dt, 0.0, 1e-300)
    assert not ok and err > 1.0
    ctx.get_state(out)
    ctx.synchronize()
    assert np.array_equal(out.cpu().numpy(), u)
    _, _, b, bh = O.dp54_tableau()
    for y0, ref, eref in ((u, u1, e1), (u1, u2, e2)):
        err, ok = ctx.step_dp54(dt, rtol, atol)
        # error-estimate parity bound (reading R29): err = rms_i(e_i / sc_i) with
        # e = dt sum_j (b_j - bh_j) k_j linear in the stage slopes k_j, each of which matches the
        # oracle to TOL * max|k_j| per variable (R20); the stage slopes of one step stay within
        # twice the first slope's scale, so |err - eref| <= max_i |de_i| / sc_i
        #   <= dt sum_j |b_j - bh_j| * 2 TOL max|f(y0)_v(i)| / sc_i,  sc_i = atol + rtol max(|y0_i|, |y_i|)
        k1 = om.rhs(y0, flux_mode=1, variant=1)[0]
        kscale = 2.0 * np.abs(k1).max(axis=(0, 2))[None, :, None]
        sc = atol + rtol * np.maximum(np.abs(y0), np.abs(ref))
        bound = dt * np.abs(b - bh).sum() * TOL * (kscale / sc).max()
        assert ok and eref <= 1.0 and abs(err - eref) <= bound, (err, eref, bound)
        ctx.get_state(out)
        ctx.synchronize()
        got = out.cpu().numpy()
        assert np.abs(got - ref).max() < 1e-13 * np.abs(ref).max()
        inc = _relerr(got - u, ref - u)
        assert (inc < 1e-10).all(), inc


@pytest.mark.parametrize("d,p", [(2, 2), (3, 3)])
def test_graph_step_bitwise_equals_eager(es, d, p):
    # es_step replays a captured CUDA graph on one rank: bitwise the eager launches, also over two
    # dt values (re-capture); es_step_host (host buffers in and out) gives the same state
    mesh, om, ctx, u = _setup(es, d, 3, p, "paper", "wave" if d == 2 else "tgv3", 1)
    ut = torch.from_numpy(u).cuda()
    out = []
    for graphs in (True, False):
        ctx.set_graphs(graphs)
        ctx.set_state(ut)
        ctx.step(1e-3, 3)
        ctx.step(5e-4, 2)
        o = torch.empty_like(ut)
        ctx.get_state(o)
        ctx.synchronize()
        out.append(o.cpu().numpy())
    assert np.array_equal(out[0], out[1])
    ctx.set_graphs(True)
    hin = torch.from_numpy(u).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ctx.step_host(hin, hout, 1e-3, 3)
    ctx.step_host(hout.clone().pin_memory(), hout, 5e-4, 2)
    assert np.array_equal(hout.numpy(), out[0])


def test_dp54_adaptive_density_wave(es):
    # adaptive DP5(4) over the density wave: reaches T; the solution matches a fine RK4 run
    mesh, om, ctx, u = _setup(es, 2, 4, 3, "paper", "wave", 1)
    T = 0.05
    ut = torch.from_numpy(u).cuda()
    ctx.set_state(ut)
    nacc, nrej, _ = ctx.integrate_dp54(T, 1e-4, rtol=1e-10, atol=1e-12)
    out = torch.empty_like(ut)
    ctx.get_state(out)
    ctx.set_state(ut)
    ctx.step(T / 400, 400)
    ref = torch.empty_like(ut)
    ctx.get_state(ref)
    ctx.synchronize()
    assert nacc >= 3
    assert (out - ref).abs().max().item() < 1e-8 * ref.abs().max().item()


def test_host_entry_point_matches_device(es):
    mesh, om, ctx, u = _setup(es, 2, 4, 4, "bj", "wave", 1)
    got = _gpu_rhs(ctx, u)
    out = np.zeros_like(u)
    ctx.rhs_host(np.ascontiguousarray(u), out)
    assert np.array_equal(out, got)  # bitwise: same kernels, same inputs
    again = _gpu_rhs(ctx, u)
    assert np.array_equal(again, got)  # deterministic


def test_inadmissible_state_flagged(es):
    L = 2.0
    mesh = I.split_cartesian(2, 3, L)
    ctx = es.Context(mesh, 2, check_admissibility=1)
    om = O.Mesh(mesh, 2)
    u = om.project(I.density_wave(om.node_coords(), L))
    u[3, 0, :] *= -1.0  # negative density in element 3
    ut = torch.from_numpy(u).cuda()
    with pytest.raises(es.ESError) as ex:
        ctx.rhs(ut, torch.empty_like(ut))
    assert ex.value.code == es.ES_ERR_INADMISSIBLE


FULL = [
    # BASELINE configs at full size, sampled elements checked against the oracle
    ("C2", 2, 32, 4, "bj", "density_wave", 1),
    ("C3", 2, 64, 10, "bj", "vortex", 1),
    ("C4", 3, 16, 4, "bj", "tgv", 0),
    ("C5", 3, 32, 8, "bj", "tgv", 1),
]


@pytest.mark.parametrize("name,d,M,p,warp,kind,fm", FULL)
def test_full_size_sampled_parity(es, name, d, M, p, warp, kind, fm):
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = _warp(warp, d, L, M)
    u = I.modal_state_from_centroids(mesh, p, kind, seed=3, amp=1e-2)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm)
    got = _gpu_rhs(ctx, u)
    ne = len(mesh["elem_vertices"])
    rng = np.random.default_rng(11)
    sample = np.unique(np.concatenate([[0, ne - 1, ne // 2], rng.integers(0, ne, 5)]))
    om = O.Mesh(mesh, p, warp=w, active=sample)
    ref, st = om.rhs(u, flux_mode=fm, variant=1, elems=sample)
    err = _relerr(got[sample], ref[sample])
    assert (err <= TOL).all(), (name, err)


def test_full_size_c4_entropy_conservation(es):
    # BASELINE C4 (EC volume and interface fluxes): sum_k w~^T M~ du~/dt = 0 to roundoff
    # (reading R21), and discrete conservation, on the full 24 576-element mesh
    d, M, p = 3, 16, 4
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    u = I.modal_state_from_centroids(mesh, p, "tgv", seed=5, amp=1e-2)
    ctx = es.Context(mesh, p, warp=I.bj_warp(d, L, M), interface_flux=0)
    rate, scale, cons = ctx.entropy_production(torch.from_numpy(u).cuda())
    assert abs(rate) <= 1e-12 * scale, (rate, scale)
    du = _gpu_rhs(ctx, u)
    assert np.abs(cons).max() <= 1e-12 * len(mesh["elem_vertices"]) * np.abs(du).max(), cons
    ctx2 = es.Context(mesh, p, warp=I.bj_warp(d, L, M), interface_flux=1)
    rate2, scale2, _ = ctx2.entropy_production(torch.from_numpy(u).cuda())
    assert rate2 < -1e-8 * scale2, (rate2, scale2)  # LLF dissipates


@pytest.mark.parametrize("d,M,p,warp,ic,fm", [(2, 3, 4, "paper", "wave", 1), (3, 3, 3, "paper", "tgv3", 1),
                                              (3, 3, 8, "bj", "tgv", 1)])
def test_eq56_ablation_parity(es, d, M, p, warp, ic, fm):
    # volume_mode 1: one flux per operator S^(l) (Eq. num_fluxes) -- same RHS as the
    # oracle's Eq. 56 path (variant 0) and as the line-wise kernel, with the Eq. 56 evaluation count
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = _warp(warp, d, L, M)
    om = O.Mesh(mesh, p, warp=w)
    u = I.perturb_modal(om.project(_ic(ic, om.node_coords(), d, L)), d, p, seed=1, amp=1e-2)
    ref, st = om.rhs(u, flux_mode=fm, variant=0)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm, volume_mode=1)
    got = _gpu_rhs(ctx, u)
    assert (_relerr(got, ref) <= TOL).all()
    c = ctx.flux_counts()
    assert c["volume"] + c["facet"] == c["eq56"]
    # kernel-counted per-operator evaluations = the Eq. 56 nonzero loops of the oracle
    cnt = ctx.count_fluxes(torch.from_numpy(u).cuda())
    assert cnt[:, 0].sum() == st.volume_pairs and cnt[:, 1].sum() == st.facet_pairs, (cnt[0], st.volume_pairs / om.ne)


@pytest.mark.parametrize("d,M,p,warp,ic,fm", [(2, 3, 3, "paper", "wave", 1), (3, 3, 2, "paper", "tgv3", 1),
                                              (3, 3, 4, "bj", "tgv", 0)])
def test_dense_ablation_parity(es, d, M, p, warp, ic, fm):
    # volume_mode 2: brute force over all node pairs with the dense operators (zeros included) --
    # the same RHS as the oracle's dense variant (2), with N_q (N_q - 1) ordered volume evaluations
    # and 2 N_q N_f N_qf facet evaluations per element
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = _warp(warp, d, L, M)
    om = O.Mesh(mesh, p, warp=w)
    u = I.perturb_modal(om.project(_ic(ic, om.node_coords(), d, L)), d, p, seed=1, amp=1e-2)
    ref, st = om.rhs(u, flux_mode=fm, variant=2)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm, volume_mode=2)
    got = _gpu_rhs(ctx, u)
    assert (_relerr(got, ref) <= TOL).all(), _relerr(got, ref)
    n = p + 1
    Nq, NF = n ** d, (d + 1) * n ** (d - 1)
    c = ctx.flux_counts()
    assert c["volume"] == Nq * (Nq - 1) and c["facet"] == 2 * Nq * NF


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2)])
def test_erk_dp8_step_parity(es, d, p):
    # es_step_erk with the Dormand-Prince 8 tableau (the paper's integrator; tools/tableaux.py)
    # against the same explicit Runge-Kutta loop over the oracle's right-hand side; and with the RK4
    # tableau against the fused RK4 path (es_step)
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import tableaux as T
    mesh, om, ctx, u = _setup(es, d, 3, p, "paper", "wave" if d == 2 else "tgv3", 1)
    dt = 2e-3
    A, b, c = T.dop853()
    ref = u.copy()
    for _ in range(2):
        ref = T.erk_step(lambda t, y: om.rhs(y, flux_mode=1, variant=1)[0], 0.0, ref, dt, A, b, c)
    ut = torch.from_numpy(u).cuda()
    ctx.set_state(ut)
    ctx.step_erk(dt, A, b, 2)
    out = torch.empty_like(ut)
    ctx.get_state(out)
    ctx.synchronize()
    got = out.cpu().numpy()
    assert np.abs(got - ref).max() < 1e-13 * np.abs(ref).max()
    assert (_relerr(got - u, ref - u) < 1e-10).all()
    A4, b4, _ = T.rk4()
    ctx.set_state(ut)
    ctx.step_erk(dt, A4, b4, 3)
    ctx.get_state(out)
    o4 = torch.empty_like(ut)
    ctx.set_state(ut)
    ctx.step(dt, 3)
    ctx.get_state(o4)
    ctx.synchronize()
    assert (_relerr(out.cpu().numpy() - u, o4.cpu().numpy() - u) < 1e-12).all()


@pytest.mark.parametrize("d,M,p,warp,ic,fm", [(2, 3, 4, "paper", "wave", 1), (2, 3, 10, "bj", "vortex", 1),
                                               (3, 3, 3, "paper", "tgv3", 1), (3, 3, 8, "bj", "tgv", 1),
                                               (3, 3, 5, "paper", "tgv3", 0)])
def test_warp_and_blend_mapping_parity(es, d, M, p, warp, ic, fm):
    """es_options.mapping_nodes = 1 (warp & blend mapping and curl-interpolation nodes, R32):
    geometry and RHS against the oracle built on its own warp & blend node set."""
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    w = _warp(warp, d, L, M)
    om = O.Mesh(mesh, p, warp=w, nodes=1)
    ctx = es.Context(mesh, p, warp=w, interface_flux=fm, mapping_nodes=1)
    for e in (0, 7, om.ne - 1):
        go, gg = om.geometry(e), ctx.element_geometry(e)
        for k in ("G", "Jn", "Jt"):
            assert np.abs(gg[k] - go[k]).max() < 1e-12 * np.abs(go[k]).max(), k
    u = om.project(_ic(ic, om.node_coords(), d, L))
    u = I.perturb_modal(u, d, p, seed=2, amp=1e-2)
    got = _gpu_rhs(ctx, u)
    ref0, _ = om.rhs(u, flux_mode=fm, variant=0)
    err = _relerr(got, ref0)
    assert (err <= TOL).all(), err
    # the lattice-node map of the same warp is a different geometry: the RHS differs
    ctx0 = es.Context(mesh, p, warp=w, interface_flux=fm, mapping_nodes=0)
    if warp != "none":
        assert np.abs(_gpu_rhs(ctx0, u) - got).max() > 1e-9 * np.abs(got).max()


@pytest.mark.parametrize("d,M,p", [(3, 12, 8), (2, 128, 10)])
def test_step_host_pipelined_bitwise(es, d, M, p):
    """es_step_host on a state above 64 MB takes the pipelined path (chunked host -> device copies
    overlapping the first stage's K1, in 3D chunked K3 + device -> host copies of the last stage): the
    same kernels on the same elements, so the state equals es_step's bit for bit, for one and for
    several steps per call."""
    L = _L(d)
    mesh = I.split_cartesian(d, M, L)
    ctx = es.Context(mesh, p, warp=I.bj_warp(d, L, M), interface_flux=1)
    u = I.modal_state_from_centroids(mesh, p, "tgv" if d == 3 else "density_wave", seed=4)
    assert u.nbytes >= 64 << 20
    ut = torch.from_numpy(u).cuda()
    dt = 2e-4 if d == 3 else 1e-5  # within the RK4 limit (2D: h = 1/64 at p = 10)
    for nsteps in (1, 2):
        ctx.set_state(ut)
        ctx.step(dt, nsteps)
        ref = torch.empty_like(ut)
        ctx.get_state(ref)
        ctx.synchronize()
        hin = torch.from_numpy(u).pin_memory()
        hout = torch.full_like(hin, float("nan")).pin_memory()
        ctx.step_host(hin, hout, dt, nsteps)
        r = ref.cpu().numpy()
        assert np.isfinite(r).all()
        assert np.array_equal(hout.numpy(), r), nsteps
