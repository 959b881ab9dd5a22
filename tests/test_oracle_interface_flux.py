"""Hand-value pins of the oracle's entropy-stable interface flux.

f*(u-, u+, n) = f#(u-, u+, n) - 1/2 lambda(u-, u+, n) (u+ - u-)         (Eq. num_flux)
lambda = max(|v- . n|, |v+ . n|) + max(sqrt(g p- / rho-), sqrt(g p+ / rho+))   (Davis)
f# = Ranocha's EC flux in direction n (P:834 with reading R3).

Every expected value below is written out by hand from those three formulas at states where f# is
trivial or short (closed forms in sqrt and log), so that the plausible mistakes named in the r01
review fail at least one case:
  * lambda instead of lambda/2 (stationary contact: mass flux doubles);
  * ||v|| instead of |v . n| (tangential velocity present);
  * the common max(|v-.n| + c-, |v+.n| + c+) instead of Davis's two separate maxima;
  * max over sides replaced by the mean or by one side's value;
  * the sign of the dissipation or of the jump (u+ - u- vs u- - u+).
"""
import math

import numpy as np
import pytest

import es_inputs as I
import oracle as O

G = 1.4


def _U(rho, v, p):
    return I.prim_to_cons(np.array([rho]), np.array([v], dtype=float), np.array([p]))[0]


def test_stationary_contact_mass_flux_is_minus_half_lambda_jump():
    # v = 0 on both sides, equal pressure, density jump: f# = (0, p n, 0) exactly,
    # lambda = 0 + max(c-, c+) = sqrt(g p / min rho), [u] = ([rho], 0, 0, 0) since E = p/(g-1)
    for d in (2, 3):
        n = np.zeros(d)
        n[0] = 1.0
        rm, rp, p = 1.0, 2.0, 1.0
        Um, Up = _U(rm, [0.0] * d, p), _U(rp, [0.0] * d, p)
        lam = math.sqrt(G * p / rm)  # = sqrt(1.4): the max is the lighter side's sound speed
        assert abs(O.wave_speed(Um, Up, n) - lam) < 1e-15
        F = O.es_flux(Um, Up, n)[0]
        expect = np.zeros(d + 2)
        expect[0] = -0.5 * lam * (rp - rm)  # = -sqrt(1.4)/2 = -0.5916079783099616
        expect[1] = p  # <p> n_1
        assert abs(expect[0] - (-0.5916079783099616)) < 1e-15
        np.testing.assert_allclose(F, expect, rtol=0, atol=2e-15)
        # the EC part alone has no mass flux: the dissipation is the whole mass flux
        Fec = O.ec_flux(Um, Up, n)[0]
        assert abs(Fec[0]) < 1e-16
        # reversing the sides reverses the jump and the mass flux sign (conservation)
        Fr = O.es_flux(Up, Um, -n)[0]
        np.testing.assert_allclose(Fr, -F, rtol=0, atol=2e-15)


def test_davis_speed_one_sided_normal_velocity_with_tangential_part():
    # u-: rho 1, v = (0.5, 0.8), p 1 -> |v.n| = 0.5, ||v|| = 0.943..., c- = sqrt(1.4)
    # u+: rho 1, v = (0, 0),     p 2 -> |v.n| = 0,   c+ = sqrt(2.8)
    # Davis: 0.5 + sqrt(2.8) = 2.17332005307; the common max(|v.n| + c) would give
    # max(0.5 + 1.1832, 1.6733) = 1.6832; ||v|| instead of |v.n| would give 0.9434 + 1.6733
    Um, Up = _U(1.0, [0.5, 0.8], 1.0), _U(1.0, [0.0, 0.0], 2.0)
    n = np.array([1.0, 0.0])
    lam = 0.5 + math.sqrt(2.8)
    assert abs(lam - 2.1733200530681511) < 1e-15
    assert abs(O.wave_speed(Um, Up, n) - lam) < 1e-15
    assert abs(O.wave_speed(Up, Um, n) - lam) < 1e-15  # symmetric in the sides
    assert abs(O.wave_speed(Um, Up, -n) - lam) < 1e-15  # |v.n| is sign-blind
    # f# by hand (R3): rho_ln = 1 (equal densities), <v>.n = 0.25, <v> = (0.25, 0.4),
    # <p> = 1.5, v-.v+ = 0, <rho/p>_ln = LM(1, 1/2) = (1/2)/ln 2 so 1/<rho/p>_ln = 2 ln 2,
    # (p- v+.n + p+ v-.n)/2 = (0 + 2 * 0.5)/2 = 0.5
    fr = 0.25
    fec = np.array([fr, fr * 0.25 + 1.5, fr * 0.4, fr * (0.0 + 2.0 * math.log(2.0) / (G - 1.0)) + 0.5])
    np.testing.assert_allclose(O.ec_flux(Um, Up, n)[0], fec, rtol=0, atol=4e-15)
    # jump [u] = u+ - u-: rho 0, rho v (-0.5, -0.8), E 2/0.4 - (1/0.4 + (0.25 + 0.64)/2) = 2.055
    jump = np.array([0.0, -0.5, -0.8, 5.0 - (2.5 + 0.445)])
    expect = fec - 0.5 * lam * jump
    np.testing.assert_allclose(O.es_flux(Um, Up, n)[0], expect, rtol=0, atol=8e-15)
    # the values spelled out: (0.25, 1.5625 + lam/4, 0.1 + 0.4 lam, 1.3664339... - 1.0275 lam)
    np.testing.assert_allclose(
        expect, [0.25, 1.5625 + 0.25 * lam, 0.1 + 0.4 * lam, 0.25 * 2 * math.log(2) / 0.4 + 0.5 - 1.0275 * lam],
        rtol=0, atol=4e-15)


def test_davis_speed_uses_separate_maxima_3d():
    # 3D, oblique unit normal; u- moves fast along n but is cold, u+ is at rest and hot
    n = np.array([1.0, 2.0, 2.0]) / 3.0
    Um = _U(2.0, [0.9, 0.3, 0.0], 0.5)   # v.n = (0.9 + 0.6)/3 = 0.5, c = sqrt(0.35)
    Up = _U(0.5, [0.0, 0.0, -0.3], 2.0)  # v.n = -0.2, c = sqrt(5.6)
    lam = 0.5 + math.sqrt(5.6)
    assert abs(O.wave_speed(Um, Up, n) - lam) < 2e-15
    # the per-side sums would give max(0.5 + 0.5916, 0.2 + 2.3664) = 2.5664 < 2.8664
    assert lam - max(0.5 + math.sqrt(0.35), 0.2 + math.sqrt(5.6)) > 0.29
    # dissipation part exactly -lam/2 [u]
    D = O.es_flux(Um, Up, n)[0] - O.ec_flux(Um, Up, n)[0]
    np.testing.assert_allclose(D, -0.5 * lam * (Up - Um), rtol=1e-14, atol=1e-14)


@pytest.mark.parametrize("d", [2, 3])
def test_dissipation_vanishes_for_equal_states_and_scales_with_jump(d):
    # f*(u, u, n) = f(u) n (consistency, P:469 + zero jump); the dissipation is linear in [u] at
    # fixed lambda: doubling a density-only jump at rest doubles the mass flux exactly
    n = np.zeros(d)
    n[-1] = 1.0
    U = _U(1.3, [0.2] * d, 0.9)
    np.testing.assert_allclose(O.es_flux(U, U, n)[0], O.euler_flux(U, n)[0], rtol=1e-14, atol=1e-14)
    U0 = _U(1.0, [0.0] * d, 1.0)
    F1 = O.es_flux(U0, _U(1.5, [0.0] * d, 1.0), n)[0]
    F2 = O.es_flux(U0, _U(2.0, [0.0] * d, 1.0), n)[0]
    # lambda = sqrt(1.4 / 1.0) in both (the lighter side is u-)
    assert abs(F1[0] - (-0.25 * math.sqrt(1.4))) < 1e-15
    assert abs(F2[0] - (-0.5 * math.sqrt(1.4))) < 1e-15
