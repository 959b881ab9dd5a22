"""Pins of the oracle's geometry and full ES modal RHS against the paper's theorems (CPU only).

- affine geometry: G = adj(grad x) exactly, J~ = det, sum w J~ = element measure
- discrete metric identities / free-stream preservation on curved meshes
- discrete conservation and entropy conservation (EC) / dissipation (ES)
- equality of the four formulations: Eq. num_fluxes loops, line-wise pairing, dense brute force,
  hybridised Chan-Wilcox eq. 35
- weight-adjusted inverse exact on affine elements
- RK4 order 4, h-convergence of order ~p+1
"""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O


def _mesh(d, M, p, warp="paper", L=None):
    L = (2.0 if d == 2 else 2 * math.pi) if L is None else L
    mesh = I.split_cartesian(d, M, L)
    w = {"paper": I.paper_warp(d, L), "bj": I.bj_warp(d, L, M), "none": None}[warp]
    return mesh, O.Mesh(mesh, p, warp=w), L


@pytest.mark.parametrize("d,p", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_affine_geometry(d, p):
    mesh, om, L = _mesh(d, 3, p, warp="none")
    W = O.ref_get(d, p, "W")
    tot = 0.0
    for e in (0, 1, 5, om.ne - 1):
        g = om.geometry(e)
        X = mesh["elem_vertex_coords"][e]
        A = ((X[1:] - X[0]) / 2.0).T  # d x / d xi for the affine map x = sum X_k lam_k
        detA = np.linalg.det(A)
        adj = detA * np.linalg.inv(A)
        assert np.abs(g["G"] - adj[None]).max() < 1e-13 * np.abs(adj).max()
        assert np.abs(g["Jt"] - detA).max() < 1e-13 * detA
        assert abs(np.sum(W * g["Jt"]) - abs(np.linalg.det(X[1:] - X[0])) / math.factorial(d)) < 1e-13
    for e in range(om.ne):
        tot += np.sum(W * om.geometry(e)["Jt"])
    assert abs(tot - L ** d) < 1e-11 * L ** d


@pytest.mark.parametrize("d,p,warp", [(2, 2, "paper"), (2, 4, "paper"), (2, 3, "bj"), (3, 2, "paper"),
                                      (3, 3, "paper"), (3, 3, "bj")])
def test_free_stream_all_variants(d, p, warp):
    mesh, om, L = _mesh(d, 3, p, warp=warp)
    u = om.project(I.free_stream(om.node_coords(), d))
    variants = [0, 1, 2, 3] if (d == 2 or p == 2) else [0, 1]
    scale = 0.0
    for e in range(om.ne):
        scale = max(scale, np.abs(om.geometry(e)["G"]).max() / om.geometry(e)["Jt"].min())
    for var in variants:
        du, st = om.rhs(u, flux_mode=1, variant=var)
        assert np.abs(du).max() < 1e-13 * scale * (p + 1) ** 2, (var, np.abs(du).max())


@pytest.mark.parametrize("d,p", [(2, 2), (2, 4), (3, 2), (3, 3)])
def test_conservation_entropy_and_variant_agreement(d, p):
    mesh, om, L = _mesh(d, 3, p, warp="paper")
    xq = om.node_coords()
    u0 = I.density_wave(xq, L) if d == 2 else I.taylor_green(xq, Ma=0.3)
    u = I.perturb_modal(om.project(u0), d, p, seed=1, amp=2e-2)
    n = p + 1
    for fm in (0, 1, 2, 3):  # EC, LLF, entropy-jump (R27) and matrix (R28) dissipation
        ref, st = om.rhs(u, flux_mode=fm, variant=0)
        # conservation and entropy balance, periodic
        cons_scale = np.abs(ref).max() * om.ne
        assert np.abs(st.conservation[:d + 2]).max() < 1e-13 * cons_scale
        if fm == 0:
            assert abs(st.entropy_rate) < 1e-12 * st.entropy_abs
        else:
            assert st.entropy_rate < -1e-6 * st.entropy_abs
        # counts: Eq. num_fluxes per element
        tens = 3 * n * n * (p + 2) // 2 if d == 2 else 4 * n ** 4
        assert st.volume_pairs + st.facet_pairs == tens * om.ne
        assert st.interface_evals == (d + 1) * (n if d == 2 else n * n) * om.ne
        vars_ = [1, 2, 3] if (d == 2 or p == 2) else [1]
        for var in vars_:
            du, st2 = om.rhs(u, flux_mode=fm, variant=var)
            assert np.abs(du - ref).max() < 2e-13 * np.abs(ref).max() * n, (fm, var)
            if var == 1:
                lw = n * n * (n + 2) if d == 2 else n ** 3 * (5 * p + 8) // 2
                assert st2.volume_pairs + st2.facet_pairs == lw * om.ne


@pytest.mark.parametrize("d,p", [(2, 3), (3, 2)])
def test_weight_adjusted_exact_on_affine(d, p):
    mesh, om, L = _mesh(d, 3, p, warp="none")
    V = O.ref_get(d, p, "V")
    W = O.ref_get(d, p, "W")
    Jt = om.geometry(2)["Jt"]
    Minv_wa = V.T @ np.diag(W / Jt) @ V  # M~^{-1} with M = I
    M = V.T @ np.diag(W * Jt) @ V
    assert np.abs(Minv_wa @ M - np.eye(len(M))).max() < 1e-13
    mesh, om2, L = _mesh(d, 3, p, warp="paper")
    Jt = om2.geometry(2)["Jt"]
    Minv_wa = V.T @ np.diag(W / Jt) @ V
    M = V.T @ np.diag(W * Jt) @ V
    assert np.abs(Minv_wa @ M - np.eye(len(M))).max() > 1e-6  # approximation on curved elements


def test_rk4_free_stream_and_order():
    mesh, om, L = _mesh(2, 3, 2, warp="paper")
    u = om.project(I.free_stream(om.node_coords(), 2))
    u1 = om.rk4(u, 1e-2, 5)
    assert np.abs(u1 - u).max() < 1e-13
    u = I.perturb_modal(om.project(I.density_wave(om.node_coords(), L)), 2, 2, seed=2, amp=1e-2)
    T = 0.08
    ref = om.rk4(u, T / 128, 128)
    errs = [np.abs(om.rk4(u, T / k, k) - ref).max() for k in (8, 16)]
    order = math.log2(errs[0] / errs[1])
    assert 3.6 < order < 4.6, order


def _rk_generic(f, y, h, n, A, b):
    """n explicit Runge-Kutta steps with tableau (A, b) -- the textbook definition"""
    s = len(b)
    for _ in range(n):
        k = []
        for i in range(s):
            k.append(f(y + h * sum(A[i, j] * k[j] for j in range(i))))
        y = y + h * sum(b[i] * k[i] for i in range(s))
    return y


def test_dp54_tableau_order():
    # Dormand-Prince 5(4) (Hairer-Norsett-Wanner I, II.5): consistency and FSAL exactly; the observed
    # convergence order on a nonlinear ODE is 5 for b and 4 for the embedded bh (a wrong coefficient
    # drops the order)
    c, A, b, bh = O.dp54_tableau()
    np.testing.assert_allclose(A.sum(1), c, atol=1e-15)
    assert abs(b.sum() - 1) < 1e-15 and abs(bh.sum() - 1) < 1e-15
    np.testing.assert_array_equal(A[6, :6], b[:6])
    for k in range(1, 6):  # quadrature conditions sum b c^(k-1) = 1/k
        assert abs(b @ c ** (k - 1) - 1.0 / k) < 1e-15
    # Lotka-Volterra; reference by scipy's DOP853 at tight tolerance
    f = lambda y: np.array([y[0] * (1 - y[1]), y[1] * (y[0] - 1)])  # noqa: E731
    from scipy.integrate import solve_ivp
    T, y0 = 2.0, np.array([1.5, 0.5])
    ref = solve_ivp(lambda t, y: f(y), (0, T), y0, method="DOP853", rtol=3e-14, atol=1e-15).y[:, -1]
    for bb, lo, hi in ((b, 4.6, 6.0), (bh, 3.6, 4.5)):
        e = [np.abs(_rk_generic(f, y0, T / n, n, A, bb) - ref).max() for n in (20, 40)]
        assert lo < math.log2(e[0] / e[1]) < hi, (lo, e)


def test_dp54_step_free_stream_and_error_scaling():
    mesh, om, L = _mesh(2, 3, 2, warp="paper")
    u = om.project(I.free_stream(om.node_coords(), 2))
    u5, err = om.dp54(u, 1e-2)
    assert np.abs(u5 - u).max() < 1e-13 and err < 1e-6
    u = I.perturb_modal(om.project(I.density_wave(om.node_coords(), L)), 2, 2, seed=2, amp=1e-2)
    # one DP5 step is much closer to a fine RK4 solution than one RK4 step; the embedded estimate
    # scales like dt^5
    dt = 0.005
    ref = om.rk4(u, dt / 32, 32)
    u5, _ = om.dp54(u, dt)
    assert np.abs(u5 - ref).max() < 0.2 * np.abs(om.rk4(u, dt, 1) - ref).max()
    e1 = om.dp54(u, dt, rtol=0.0, atol=1.0)[1]
    e2 = om.dp54(u, dt / 2, rtol=0.0, atol=1.0)[1]
    assert 4.3 < math.log2(e1 / e2) < 5.7, (e1, e2)


def _l2_density_error(om, u, L, t, d):
    V = O.ref_get(d, om.p, "V")
    W = O.ref_get(d, om.p, "W")
    err = 0.0
    for e in range(om.ne):
        g = om.geometry(e)
        rho = V @ u[e, 0]
        x = g["xq"] - t
        rho_ex = 1.0 + 0.2 * np.sin(2 * math.pi / L * np.sum(x, axis=1))
        err += np.sum(W * g["Jt"] * (rho - rho_ex) ** 2)
    return math.sqrt(err)


def test_density_wave_h_convergence():
    # ES scheme, density wave translating with v = (1,1) over one period T = 2 on the
    # paper's curved triangles, p = 3: the observed order at M = 8 -> 16 is within 0.3 of p + 1
    # (the GPU study in profiles/r02_density_wave_convergence.jsonl measures 3.81 there with
    # the degree-35 rule)
    d, p, L, T = 2, 3, 2.0, 2.0
    errs = []
    for M in (8, 16):
        mesh, om, _ = _mesh(d, M, p, warp="paper")
        u = om.project(I.density_wave(om.node_coords(), L))
        h = L / M
        nst = int(math.ceil(T / (0.1 * h / ((2 * p + 1) * 3.05))))  # CFL 0.1 (R16)
        u = om.rk4(u, T / nst, nst, flux_mode=1)
        errs.append(_l2_density_error(om, u, L, T, d))
    order = math.log2(errs[0] / errs[1])
    assert abs(order - (p + 1)) <= 0.3, (errs, order)
