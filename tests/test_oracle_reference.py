"""Pins of the oracle's 1D rules, reference SBP operators and PKD basis (CPU only).

Each test pins the oracle to something other than itself: closed forms, scipy's independent
Gauss-Jacobi routine, polynomial exactness, the SBP property, the facet decomposition
(P:131), printed/derived counts and orthonormality.
"""
import itertools
import math

import numpy as np
import pytest
from scipy.special import roots_jacobi

import oracle as O


# ---------------------------------------------------------------- 1D
def test_gauss_closed_forms(golden):
    g = golden["gauss_rules"]
    for key, (q, a) in {"q0_00": (0, 0), "q1_00": (1, 0), "q0_10": (0, 1)}.items():
        x, w = O.gauss_jacobi(q, a, 0)
        np.testing.assert_allclose(x, g[key]["x"], atol=1e-15)
        np.testing.assert_allclose(w, g[key]["w"], atol=1e-15)


@pytest.mark.parametrize("a", [0, 1])
@pytest.mark.parametrize("q", [2, 3, 5, 8, 10, 12])
def test_gauss_vs_scipy_and_exactness(q, a):
    x, w = O.gauss_jacobi(q, a, 0)
    xr, wr = roots_jacobi(q + 1, a, 0)  # independent library routine
    np.testing.assert_allclose(x, xr, atol=2e-15)
    np.testing.assert_allclose(w, wr, rtol=1e-13, atol=1e-15)
    # exact for degree 2q+1 against the weight (1-x)^a (delta = 1)
    for k in range(2 * q + 2):
        # int_{-1}^1 x^k (1-x)^a dx in closed form
        exact = (1 - (-1) ** (k + 1)) / (k + 1) if a == 0 else \
            (1 - (-1) ** (k + 1)) / (k + 1) - (1 - (-1) ** (k + 2)) / (k + 2)
        assert abs(np.sum(w * x ** k) - exact) < 1e-13
    # not exact at degree 2q+2 (it is a Gauss rule, not more)
    k = 2 * q + 2
    exact = (1 - (-1) ** (k + 1)) / (k + 1) if a == 0 else \
        (1 - (-1) ** (k + 1)) / (k + 1) - (1 - (-1) ** (k + 2)) / (k + 2)
    assert abs(np.sum(w * x ** k) - exact) > 1e-10


def test_jacobi_values_orthonormality_derivative(golden):
    for v in golden["jacobi_values"][:-1]:
        assert abs(O.jacobi(v["n"], v["a"], v["b"], v["x"]) - v["v"]) < 1e-15
    for a in (0, 1, 3, 7):
        x, w = roots_jacobi(14, a, 0)  # independent rule, exact to degree 27
        P = np.array([[O.jacobi(i, a, 0, xx) for xx in x] for i in range(13)])
        np.testing.assert_allclose(P @ np.diag(w) @ P.T, np.eye(13), atol=1e-12)
        for n in range(0, 12):
            for xx in np.linspace(-0.9, 0.9, 7):
                h = 1e-6
                fd = (O.jacobi(n, a, 0, xx + h) - O.jacobi(n, a, 0, xx - h)) / (2 * h)
                assert abs(fd - O.jacobi_deriv(n, a, 0, xx)) < 1e-6 * max(1, abs(fd))


def test_lagrange_diff():
    np.testing.assert_allclose(O.lagrange_diff([-1.0, 1.0]), [[-0.5, 0.5], [-0.5, 0.5]], atol=1e-16)
    x, _ = O.gauss_jacobi(6, 0, 0)
    D = O.lagrange_diff(x)
    for k in range(7):
        np.testing.assert_allclose(D @ x ** k, k * x ** max(k - 1, 0) if k else 0 * x, atol=1e-12)


# ---------------------------------------------------------------- reference operators
def _monomials(d, deg):
    return [m for m in itertools.product(range(deg + 1), repeat=d) if sum(m) <= deg]


@pytest.mark.parametrize("d,q", [(2, 1), (2, 2), (2, 4), (2, 7), (2, 10), (3, 1), (3, 2), (3, 3), (3, 5)])
def test_sbp_operators(d, q, golden):
    Q = O.ref_get(d, q, "Q")
    E = O.ref_get(d, q, "E")
    S = O.ref_get(d, q, "S")
    D = O.ref_get(d, q, "D")
    R = O.ref_get(d, q, "R")
    W = O.ref_get(d, q, "W")
    B = O.ref_get(d, q, "B")
    xi = O.ref_get(d, q, "xi")
    xif = O.ref_get(d, q, "xif")
    nh = O.ref_get(d, q, "nhat")
    tol = 1e-12 if d == 2 else 1e-11
    # SBP property Q + Q^T = E with E from the facet decomposition
    for m in range(d):
        assert np.abs(Q[m] + Q[m].T - E[m]).max() < tol
        assert np.abs(S[m] + S[m].T).max() < tol          # skew part
        assert np.abs(np.diag(S[m])).max() < tol
    # reference measure
    meas = golden["reference_measure"]["tri" if d == 2 else "tet"]
    assert abs(W.sum() - meas) < 1e-13 and (W > 0).all()
    # D exact on P_q, R exact on P_q, E integrates u v n_m exactly for u v in P_2q
    for mono in _monomials(d, q):
        v = np.prod(xi ** np.array(mono), axis=1)
        for m in range(d):
            dm = np.array(mono)
            c = dm[m]
            dm[m] = max(c - 1, 0)
            dv = c * np.prod(xi ** dm, axis=1) if c else 0 * v
            assert np.abs(D[m] @ v - dv).max() < 1e-9 * max(1, np.abs(dv).max())
        for z in range(d + 1):
            assert np.abs(R[z] @ v - np.prod(xif[z] ** np.array(mono), axis=1)).max() < 1e-10
    # volume quadrature exact to degree 2q-1; facet rules exact for the facet integral:
    # sum_z nhat_m 1^T B 1 = int n_m ds = 0 (closed surface), |facet 2| weights carry sqrt2/sqrt3
    for m in range(d):
        assert abs(sum(nh[z, m] * B[z].sum() for z in range(d + 1))) < 1e-13


def _simplex_monomial_integral(mono):
    # int over the reference simplex {xi >= -1, sum xi <= -1 + ... } via substitution xi = -1 + 2 lam
    # int lam^a over the unit simplex = prod a_i! / (d + sum a)!  (Dirichlet integral)
    d = len(mono)
    tot = 0.0
    # expand prod (-1 + 2 lam_i)^{m_i}
    for ks in itertools.product(*[range(m + 1) for m in mono]):
        coef = 1.0
        for m, k in zip(mono, ks):
            coef *= math.comb(m, k) * (2.0 ** k) * ((-1.0) ** (m - k))
        num = math.prod(math.factorial(k) for k in ks)
        tot += coef * num / math.factorial(d + sum(ks))
    return tot * 2.0 ** d


@pytest.mark.parametrize("d,q", [(2, 2), (2, 5), (3, 2), (3, 4)])
def test_volume_quadrature_exactness(d, q):
    W = O.ref_get(d, q, "W")
    xi = O.ref_get(d, q, "xi")
    for mono in _monomials(d, 2 * q - 1):
        val = np.sum(W * np.prod(xi ** np.array(mono), axis=1))
        assert abs(val - _simplex_monomial_integral(mono)) < 1e-12


def test_collapsed_map_tet(golden):
    # reading R1: corrected map; the centre of the eta-cube maps to (-0.75,-0.5,0)
    xi = O.ref_get(3, 0, "xi")  # q = 0: single node at eta = (0, 0, -1/3)
    eta = O.ref_get(3, 0, "eta")
    e1, e2, e3 = eta[0]
    assert abs(xi[0, 0] - (0.25 * (1 + e1) * (1 - e2) * (1 - e3) - 1)) < 1e-15
    g = golden["collapsed_map_tet_origin"]
    # evaluate the same map at eta = 0 through the q=0 node formula with eta3 = 0
    x0 = 0.25 * (1 + 0) * (1 - 0) * (1 - 0) - 1
    assert (x0, 0.5 * (1 + 0) * (1 - 0) - 1, 0.0) == tuple(g["xi"])


def _eq56_count(d, q):
    S = O.ref_get(d, q, "S")
    R = O.ref_get(d, q, "R")
    B = O.ref_get(d, q, "B")
    vol = sum(int(np.sum(np.abs(S[l]) > 1e-12 * np.abs(S[l]).max())) // 2 for l in range(d))
    fac = 0
    for z in range(d + 1):
        RB = R[z].T * B[z][None, :]
        fac += int(np.sum(np.abs(RB) > 1e-12 * np.abs(RB).max()))
    return vol, fac


@pytest.mark.parametrize("d,q", [(2, 1), (2, 2), (2, 3), (2, 5), (2, 10), (3, 1), (3, 2), (3, 3), (3, 5)])
def test_flux_counts_closed_forms(d, q):
    vol, fac = _eq56_count(d, q)
    n = q + 1
    if d == 2:
        assert vol + fac == 3 * n * n * (q + 2) // 2
        assert fac == 3 * n * n
    else:
        assert vol + fac == 4 * n ** 4
        assert fac == 3 * n ** 3 + n ** 4


def test_flux_count_paper_ratios(golden):
    md = golden["multidim_node_counts"]
    for d, key in ((2, "flux_count_ratio_tri"), (3, "flux_count_ratio_tet")):
        for q, ratio in zip(golden[key]["q"], golden[key]["ratio"]):
            if d == 3 and q == 10:
                tens = 4 * (q + 1) ** 4  # closed form, pinned above for q <= 5
            elif d == 2 and q == 10:
                tens = sum(_eq56_count(d, q))
            else:
                tens = sum(_eq56_count(d, q))
            if d == 2:
                Nv, Nf_nodes, Nf = md["tri_volume"][str(q)], q + 1, 3
            else:
                Nv, Nf_nodes, Nf = md["tet_volume"][str(q)], md["tet_facet"][str(q)], 4
            multi = d * Nv * (Nv - 1) // 2 + Nf * Nv * Nf_nodes
            assert abs(multi / tens - ratio) < 0.006, (d, q, multi / tens, ratio)
    assert sum(_eq56_count(2, 2)) == golden["tensor_counts"]["tri_q2"]
    assert sum(_eq56_count(3, 2)) == golden["tensor_counts"]["tet_q2"]
    assert _eq56_count(2, 2)[0] == golden["tensor_counts"]["tri_q2_volume"]


# ---------------------------------------------------------------- PKD basis
@pytest.mark.parametrize("d,p", [(2, 1), (2, 2), (2, 4), (2, 10), (3, 2), (3, 3), (3, 4), (3, 8)])
def test_pkd_orthonormal(d, p):
    V = O.ref_get(d, p, "V")
    W = O.ref_get(d, p, "W")
    assert np.abs(V.T @ np.diag(W) @ V - np.eye(V.shape[1])).max() < 5e-14 * p * p
    # homogenised Cartesian evaluation == principal-function product at the nodes
    xi = O.ref_get(d, p, "xi")
    vals, grads = O.pkd_eval(d, p, xi)
    assert np.abs(vals - V).max() < 1e-12 * max(1, np.abs(V).max())


def test_pkd_constant_mode_and_shapes(golden):
    V = O.ref_get(2, 2, "V")
    assert V.shape == tuple(golden["vandermonde_shapes"]["tri_p2"])
    assert np.abs(V[:, 0] - golden["pkd_constant_mode_tri"]["value"]).max() < 1e-15
    V3 = O.ref_get(3, 3, "V")
    assert V3.shape == tuple(golden["vandermonde_shapes"]["tet_p3"])
    assert np.abs(V3[:, 0] - math.sqrt(3.0 / 4.0)).max() < 1e-14  # 1/sqrt(|tet| = 4/3)


@pytest.mark.parametrize("d,p", [(2, 4), (3, 3)])
def test_pkd_gradient_fd_and_vertices(d, p):
    rng = np.random.default_rng(0)
    pts = []
    while len(pts) < 6:
        x = rng.uniform(-1, 1, d)
        if x.sum() <= -1 + (d == 2) * 1.0 - 0.05:
            pts.append(x)
    pts = np.array(pts)
    v, g = O.pkd_eval(d, p, pts)
    h = 1e-6
    for k in range(d):
        e = np.zeros(d)
        e[k] = h
        vp, _ = O.pkd_eval(d, p, pts + e)
        vm, _ = O.pkd_eval(d, p, pts - e)
        assert np.abs((vp - vm) / (2 * h) - g[:, :, k]).max() < 1e-6
    # finite at the collapsed vertex (the homogenised form has no singularity)
    top = np.array([[-1.0, 1.0]]) if d == 2 else np.array([[-1.0, -1.0, 1.0]])
    v, g = O.pkd_eval(d, p, top)
    assert np.isfinite(v).all() and np.isfinite(g).all()
