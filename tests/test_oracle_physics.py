"""Pins of the oracle's Euler physics (readings R3, R5, R7)."""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O

G = 1.4


def _prim(U):
    d = U.shape[-1] - 2
    rho = U[..., 0]
    v = U[..., 1:1 + d] / rho[..., None]
    p = (G - 1) * (U[..., -1] - 0.5 * rho * np.sum(v * v, -1))
    return rho, v, p


def test_printed_examples(golden):
    ex = golden["euler_flux_example"]
    U = I.prim_to_cons(np.array([1.0]), np.array([[1.0, 0.0]]), np.array([1.0]))
    F = O.euler_flux(U, [1.0, 0.0])
    np.testing.assert_allclose(F[0], ex["F"], atol=1e-15)
    U = I.prim_to_cons(np.array([1.0]), np.array([[0.0, 0.0]]), np.array([golden["entropy_example"]["p"]]))
    S, Fe = O.entropy(U)
    assert abs(S[0] - golden["entropy_example"]["S"]) < 1e-14
    U = I.prim_to_cons(np.array([2.0]), np.array([[0.3, -0.2]]), np.array([4.0]))
    assert abs(O.entropy_vars(U)[0, -1] - golden["w_last_example"]["w_last"]) < 1e-15
    for ex in golden["log_mean_examples"][:-1]:
        assert abs(O.ln_mean(ex["x"], ex["y"]) - ex["v"]) < 2e-15 * ex["v"]
        assert abs(O.inv_ln_mean(ex["x"], ex["y"]) * ex["v"] - 1) < 2e-15
    U = I.prim_to_cons(np.array([1.0]), np.array([[0.0, 0.0]]), np.array([1.0]))
    assert abs(O.wave_speed(U[0], U[0], np.array([1.0, 0.0])) - golden["wave_speed_rest"]["value"]) < 1e-15


def test_log_mean_branches():
    # series branch near x = y vs a 50-digit evaluation of (y-x)/ln(y/x) through log1p
    for x, y in [(1.0, 1.0 + 1e-3), (0.3, 0.3001), (5.0, 5.002), (1.0, 1.0199)]:
        t = (y - x) / x
        exact = (y - x) / math.log1p(t)
        assert abs(O.ln_mean(x, y) - exact) < 3e-16 * exact
        assert abs(O.inv_ln_mean(x, y) * exact - 1) < 3e-16
    # symmetric
    assert O.ln_mean(2.0, 3.0) == O.ln_mean(3.0, 2.0) or abs(O.ln_mean(2.0, 3.0) - O.ln_mean(3.0, 2.0)) < 1e-15


@pytest.mark.parametrize("d", [2, 3])
def test_entropy_variables(d):
    U = I.random_states(200, d, seed=1)
    W = O.entropy_vars(U)
    np.testing.assert_allclose(O.cons_from_entropy(W), U, rtol=1e-13, atol=1e-13)
    # W = grad_U S by central differences (S = -rho ln(p/rho^g)/(g-1))
    h = 1e-6
    for i in range(0, 200, 40):
        for k in range(d + 2):
            e = np.zeros(d + 2)
            e[k] = h * max(1.0, abs(U[i, k]))
            Sp, _ = O.entropy(U[i] + e)
            Sm, _ = O.entropy(U[i] - e)
            assert abs((Sp[0] - Sm[0]) / (2 * e[k]) - W[i, k]) < 1e-7


@pytest.mark.parametrize("d", [2, 3])
def test_ec_flux_consistency_symmetry_tadmor(d):
    Ua = I.random_states(500, d, seed=2, spread=0.6)
    Ub = I.random_states(500, d, seed=3, spread=0.6)
    rng = np.random.default_rng(4)
    nv = rng.standard_normal((500, d))
    # consistency f#(U,U,n) = f(U,n)
    np.testing.assert_allclose(O.ec_flux(Ua, Ua, nv), O.euler_flux(Ua, nv), rtol=1e-14, atol=1e-13)
    # symmetry
    np.testing.assert_allclose(O.ec_flux(Ua, Ub, nv), O.ec_flux(Ub, Ua, nv), rtol=1e-14, atol=1e-14)
    # Tadmor's condition in directional form with psi_m = rho v_m
    Wa, Wb = O.entropy_vars(Ua), O.entropy_vars(Ub)
    F = O.ec_flux(Ua, Ub, nv)
    psi_a = np.sum(Ua[:, 1:1 + d] * nv, 1)
    psi_b = np.sum(Ub[:, 1:1 + d] * nv, 1)
    res = np.sum((Wb - Wa) * F, 1) - (psi_b - psi_a)
    scale = np.sum(np.abs(Wb - Wa) * np.abs(F), 1) + 1
    assert np.abs(res / scale).max() < 1e-13
    # the energy component as printed at P:834 (1/2 multiplying both terms) fails consistency (R3)
    rho, v, p = _prim(Ua)
    vn = np.sum(v * nv, 1)
    printed = 0.5 * rho * vn * (np.sum(v * v, 1) + p / rho / (G - 1)) + p * vn
    assert np.abs(printed - O.euler_flux(Ua, nv)[:, -1]).max() > 1e-2


@pytest.mark.parametrize("d", [2, 3])
def test_dudw_is_the_inverse_entropy_hessian(d):
    # R27: du/dw in closed form against central differences of the paper's map u(w) (R7)
    # and of w(u); symmetric positive definite
    U = I.random_states(40, d, seed=11, spread=0.6)
    A = O.dudw(U)
    W = O.entropy_vars(U)
    h = 1e-6
    for i in range(0, 40, 8):
        Jw = np.zeros((d + 2, d + 2))
        Ju = np.zeros((d + 2, d + 2))
        for k in range(d + 2):
            e = np.zeros(d + 2)
            e[k] = h * max(1.0, abs(W[i, k]))
            Jw[:, k] = (O.cons_from_entropy(W[i] + e)[0] - O.cons_from_entropy(W[i] - e)[0]) / (2 * e[k])
            e = np.zeros(d + 2)
            e[k] = h * max(1.0, abs(U[i, k]))
            Ju[:, k] = (O.entropy_vars(U[i] + e)[0] - O.entropy_vars(U[i] - e)[0]) / (2 * e[k])
        assert np.abs(A[i] - Jw).max() < 1e-7 * np.abs(A[i]).max()
        assert np.abs(A[i] @ Ju - np.eye(d + 2)).max() < 1e-6
        np.testing.assert_allclose(A[i], A[i].T, rtol=1e-15, atol=1e-15)
        assert np.linalg.eigvalsh(A[i]).min() > 0


@pytest.mark.parametrize("d", [2, 3])
def test_entropy_jump_flux(d):
    # interface flux mode 2 (R27): consistent, conservative, entropy stable with the exact
    # dissipation -lambda/2 [w]^T (du/dw) [w], and equal to local Lax-Friedrichs to O(|[u]|^2)
    Ua = I.random_states(300, d, seed=12, spread=0.6)
    Ub = I.random_states(300, d, seed=13, spread=0.6)
    rng = np.random.default_rng(14)
    n = rng.standard_normal((300, d))
    n /= np.linalg.norm(n, axis=1)[:, None]
    F = O.ej_flux(Ua, Ub, n)
    np.testing.assert_allclose(O.ej_flux(Ua, Ua, n), O.euler_flux(Ua, n), rtol=1e-14, atol=1e-13)
    np.testing.assert_allclose(F, -O.ej_flux(Ub, Ua, -n), rtol=1e-13, atol=1e-13)
    Wa, Wb = O.entropy_vars(Ua), O.entropy_vars(Ub)
    dw = Wb - Wa
    lhs = np.sum(dw * F, 1)
    rhs = np.sum(Ub[:, 1:1 + d] * n, 1) - np.sum(Ua[:, 1:1 + d] * n, 1)
    assert (lhs - rhs < 0).all()  # P:488, strictly for distinct states
    # the dissipation as stated, with du/dw at u(wbar) and Davis's speed
    Um = O.cons_from_entropy(0.5 * (Wa + Wb))
    A = O.dudw(Um)
    lam = np.array([O.wave_speed(Ua[i], Ub[i], n[i]) for i in range(300)])
    Dexp = -0.5 * lam[:, None] * np.einsum("nij,nj->ni", A, dw)
    np.testing.assert_allclose(F - O.ec_flux(Ua, Ub, n), Dexp, rtol=1e-12, atol=1e-12)
    # small jumps: (du/dw)[w] = [u] + O(|[u]|^2), so the flux approaches local Lax-Friedrichs
    errs = []
    for eps in (1e-2, 5e-3):
        Uc = Ua[:20] * (1.0 + eps * rng.standard_normal((20, d + 2)) * 0.1)
        errs.append(np.abs(O.ej_flux(Ua[:20], Uc, n[:20]) - O.es_flux(Ua[:20], Uc, n[:20])).max())
    assert errs[0] < 1e-3 and errs[1] < errs[0] / 2.5


@pytest.mark.parametrize("d", [2, 3])
def test_matrix_dissipation_flux(d):
    # interface flux mode 3 (R28): f* - f# = -1/2 |A_n| (du/dw) [w] at U(wbar), with |A_n| from
    # numpy's eigendecomposition of a finite-difference Jacobian of the normal Euler flux
    Ua = I.random_states(60, d, seed=15, spread=0.6)
    Ub = I.random_states(60, d, seed=16, spread=0.6)
    rng = np.random.default_rng(17)
    n = rng.standard_normal((60, d))
    n /= np.linalg.norm(n, axis=1)[:, None]
    F = O.md_flux(Ua, Ub, n)
    Wa, Wb = O.entropy_vars(Ua), O.entropy_vars(Ub)
    Um = O.cons_from_entropy(0.5 * (Wa + Wb))
    A0 = O.dudw(Um)
    for i in range(0, 60, 6):
        J = np.zeros((d + 2, d + 2))
        for k in range(d + 2):
            e = np.zeros(d + 2)
            e[k] = 1e-6 * max(1.0, abs(Um[i, k]))
            J[:, k] = (O.euler_flux(Um[i] + e, n[i])[0] - O.euler_flux(Um[i] - e, n[i])[0]) / (2 * e[k])
        lam, R = np.linalg.eig(J)
        absA = (R @ np.diag(np.abs(lam)) @ np.linalg.inv(R)).real
        D = -0.5 * absA @ A0[i] @ (Wb[i] - Wa[i])
        np.testing.assert_allclose(F[i] - O.ec_flux(Ua[i], Ub[i], n[i])[0], D, rtol=1e-7, atol=1e-8 * np.abs(F[i]).max())
    np.testing.assert_allclose(O.md_flux(Ua, Ua, n), O.euler_flux(Ua, n), rtol=1e-14, atol=1e-13)
    np.testing.assert_allclose(F, -O.md_flux(Ub, Ua, -n), rtol=1e-13, atol=1e-13)
    lhs = np.sum((Wb - Wa) * F, 1)
    rhs = np.sum(Ub[:, 1:1 + d] * n, 1) - np.sum(Ua[:, 1:1 + d] * n, 1)
    assert (lhs - rhs < 0).all()  # |A_n| du/dw is symmetric positive semi-definite


@pytest.mark.parametrize("d", [2, 3])
def test_es_flux_conservation_and_entropy_condition(d):
    Ua = I.random_states(300, d, seed=5, spread=0.6)
    Ub = I.random_states(300, d, seed=6, spread=0.6)
    rng = np.random.default_rng(7)
    n = rng.standard_normal((300, d))
    n /= np.linalg.norm(n, axis=1)[:, None]
    Fab = O.es_flux(Ua, Ub, n)
    Fba = O.es_flux(Ub, Ua, -n)
    np.testing.assert_allclose(Fab, -Fba, rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(O.es_flux(Ua, Ua, n), O.euler_flux(Ua, n), rtol=1e-14, atol=1e-13)
    Wa, Wb = O.entropy_vars(Ua), O.entropy_vars(Ub)
    lhs = np.sum((Wb - Wa) * Fab, 1)
    rhs = np.sum(Ub[:, 1:1 + d] * n, 1) - np.sum(Ua[:, 1:1 + d] * n, 1)
    assert (lhs - rhs <= 1e-12).all()  # P:488 entropy condition
    # Davis wave speed is an upper bound of |v.n| + c on both sides
    for i in range(20):
        lam = O.wave_speed(Ua[i], Ub[i], n[i])
        for U in (Ua[i], Ub[i]):
            rho, v, p = _prim(U[None])
            assert lam >= abs(v[0] @ n[i]) + math.sqrt(G * p[0] / rho[0]) - 1e-14


def test_initial_conditions(golden):
    g = golden["ic_density_wave"]
    U = I.density_wave(np.array([g[0]["x"], g[1]["x"]]), L=2.0)
    assert abs(U[0, 0] - 1.0) < 1e-15 and abs(U[0, -1] - g[0]["E"]) < 1e-14
    assert abs(U[1, 0] - g[1]["rho"]) < 1e-14
    t = golden["ic_tgv"]
    U = I.taylor_green(np.array([t["x"]]), Ma=t["Ma"])
    rho, v, p = _prim(U)
    np.testing.assert_allclose(v[0], t["v"], atol=1e-15)
    assert abs(p[0] - t["p"]) < 1e-10
