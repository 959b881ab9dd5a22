"""CPU checks of the product's host setup (no GPU): the reference tables the kernels use, compared
against the oracle's dense operators.  This pins the line factorisation the kernels rely on
(DESIGN.md 5.3): on an eta_k line, S^(l)_ij = c_k,l(line) * skew(X_k,l)[a_i, a_j]."""
import numpy as np
import pytest

import oracle as O


@pytest.fixture(scope="module")
def es():
    from tools.build import build_lib
    build_lib()
    import paper_2312_07874_b200 as es
    return es


CASES = [(2, 1), (2, 2), (2, 3), (2, 4), (2, 7), (2, 10), (3, 1), (3, 2), (3, 3), (3, 4), (3, 5)]


def _ulps(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.abs(a - b) / np.maximum(np.spacing(np.abs(b)), np.spacing(1.0) * 1e-3)


@pytest.mark.parametrize("d,p", CASES)
def test_rules_weights_nodes(es, d, p):
    eta, w = O.gauss_jacobi(p, 0, 0)
    e3, w3 = O.gauss_jacobi(p, 1, 0)
    for name, ref in (("eta", eta), ("w", w), ("eta3", e3), ("w3", w3)):
        got = es.ref_table(d, p, name)
        assert np.all((_ulps(got, ref) <= 2) | (np.abs(got - ref) < 1e-18)), name
    W = O.ref_get(d, p, "W")
    assert _ulps(es.ref_table(d, p, "Wvol"), W).max() <= 2
    B = O.ref_get(d, p, "B")
    assert _ulps(es.ref_table(d, p, "Bf"), B.ravel()).max() <= 2
    xi = O.ref_get(d, p, "xi")
    assert np.abs(es.ref_table(d, p, "xi_vol") - xi.ravel()).max() < 4e-16


def _lines(d, n, k, diagonal=False):
    """node index pairs (i, j, pos_i, pos_j, fixed coords) along eta_k lines"""
    import itertools
    out = []
    for fixed in itertools.product(range(n), repeat=d - 1):
        for a in range(n):
            for b in range(n):
                if a == b and not diagonal:
                    continue
                ci, cj, it = [0] * d, [0] * d, iter(fixed)
                for t in range(d):
                    if t == k:
                        ci[t], cj[t] = a, b
                    else:
                        ci[t] = cj[t] = next(it)
                i = sum(ci[t] * n ** t for t in range(d))
                j = sum(cj[t] * n ** t for t in range(d))
                out.append((i, j, a, b, ci))
    return out


@pytest.mark.parametrize("d,p", CASES)
def test_line_factorisation_matches_dense_S(es, d, p):
    n = p + 1
    S = O.ref_get(d, p, "S")
    w = es.ref_table(d, p, "w")
    w3 = es.ref_table(d, p, "w3")
    eta = es.ref_table(d, p, "eta")
    sk = {nm: es.ref_table(d, p, nm).reshape(n, n) for nm in ("skQ1", "skA1", "skA2")}
    if d == 3:
        sk.update({nm: es.ref_table(d, p, nm).reshape(n, n) for nm in ("skA3", "skA4")})
    scale = np.abs(S).max()
    for k in range(d):
        for i, j, a, b, c in _lines(d, n, k):
            if d == 2:
                if k == 0:
                    expect = [w[c[1]] * sk["skQ1"][a, b], w[c[1]] * sk["skA1"][a, b]]
                else:
                    expect = [0.0, w[c[0]] * sk["skA2"][a, b]]
            else:
                if k == 0:
                    cl = 0.5 * w[c[1]] * w3[c[2]]
                    expect = [cl * sk["skQ1"][a, b], cl * sk["skA1"][a, b], cl * sk["skA1"][a, b]]
                elif k == 1:
                    cl = 0.5 * w[c[0]] * w3[c[2]]
                    expect = [0.0, cl * sk["skA2"][a, b], cl * sk["skA3"][a, b]]
                else:
                    cl = 0.125 * w[c[0]] * w[c[1]] * (1 - eta[c[1]])
                    expect = [0.0, 0.0, cl * sk["skA4"][a, b]]
            for l in range(d):
                assert abs(S[l, i, j] - expect[l]) < 1e-14 * scale, (k, l, i, j)
    # and S has no entries off the lines
    mask = np.zeros_like(S[0], dtype=bool)
    for k in range(d):
        for i, j, *_ in _lines(d, n, k):
            mask[i, j] = True
    for l in range(d):
        assert np.abs(S[l][~mask]).max() < 1e-14 * scale


@pytest.mark.parametrize("d,p", CASES)
def test_line_factorisation_matches_dense_Q(es, d, p):
    # Q^(l) = W D^(l) is the sum over line directions of coefficient x X with
    # the unskewed 1D matrices (the linear-advection workload's skew-symmetric form uses Q itself)
    n = p + 1
    Qd = O.ref_get(d, p, "Q")
    w = es.ref_table(d, p, "w")
    w3 = es.ref_table(d, p, "w3")
    eta = es.ref_table(d, p, "eta")
    X = {nm: es.ref_table(d, p, nm).reshape(n, n) for nm in ("fQ1", "fA1", "fA2")}
    if d == 3:
        X.update({nm: es.ref_table(d, p, nm).reshape(n, n) for nm in ("fA3", "fA4")})
    Qa = np.zeros_like(Qd)
    for k in range(d):
        for i, j, a, b, c in _lines(d, n, k, diagonal=True):
            if d == 2:
                ex = [w[c[1]] * X["fQ1"][a, b], w[c[1]] * X["fA1"][a, b]] if k == 0 else [0.0, w[c[0]] * X["fA2"][a, b]]
            elif k == 0:
                cl = 0.5 * w[c[1]] * w3[c[2]]
                ex = [cl * X["fQ1"][a, b], cl * X["fA1"][a, b], cl * X["fA1"][a, b]]
            elif k == 1:
                cl = 0.5 * w[c[0]] * w3[c[2]]
                ex = [0.0, cl * X["fA2"][a, b], cl * X["fA3"][a, b]]
            else:
                cl = 0.125 * w[c[0]] * w[c[1]] * (1 - eta[c[1]])
                ex = [0.0, 0.0, cl * X["fA4"][a, b]]
            for l in range(d):
                Qa[l, i, j] += ex[l]
    assert np.abs(Qa - Qd).max() < 2e-14 * np.abs(Qd).max()


@pytest.mark.parametrize("d,p", [(2, 3), (2, 6), (3, 2), (3, 4)])
def test_extrapolation_and_pkd_tables(es, d, p):
    n = p + 1
    R = O.ref_get(d, p, "R")
    lL, lR = es.ref_table(d, p, "lL"), es.ref_table(d, p, "lR")
    # facet 2 (eta1 = +1): R^(2) row of facet node (b[,c]) is lR along the eta1 line
    f = 1
    if d == 2:
        i0 = f * n
        np.testing.assert_allclose(R[1, f, i0:i0 + n], lR, atol=1e-15)
        np.testing.assert_allclose(R[0, f, f::n], lL, atol=1e-15)
    else:
        l3 = es.ref_table(d, p, "l3L")
        li4 = es.ref_table(d, p, "lint4").reshape(n, n)
        np.testing.assert_allclose(R[1, f, f * n:f * n + n], lR, atol=1e-15)
        # facet 4 node (a=0, j=1): R = l_b(eta3_j) l3_c(-1) over the (b, c) plane of a = 0
        row = R[3, 0 + n * 1].reshape(n, n, n)[:, :, 0]  # [c][b]
        np.testing.assert_allclose(row, np.outer(l3, li4[1]), atol=1e-14)
    V = O.ref_get(d, p, "V")
    p1 = es.ref_table(d, p, "psi1").reshape(n, n)
    p2 = es.ref_table(d, p, "psi2").reshape(n, n, n)
    p3 = es.ref_table(d, p, "psi3").reshape(n, n, n)
    al = O.ref_get(d, p, "alpha").astype(int)
    for k, a in enumerate(al):
        for i in range(V.shape[0]):
            A, B_, C = i % n, (i // n) % n, i // (n * n)
            v = p1[a[0], A] * p2[a[0], a[1], B_]
            if d == 3:
                v *= p3[a[0] + a[1], a[2], C]
            assert abs(v - V[i, k]) < 1e-14 * max(1.0, abs(V[i, k]))


@pytest.mark.parametrize("d,N", [(2, 3), (2, 8), (2, 11), (3, 3), (3, 6), (3, 9)])
def test_warp_and_blend_nodes_match_oracle(es, d, N):
    """The product's warp & blend mapping nodes (binary128, Gauss-Jacobi (1,1) interior GLL points,
    barycentric Lagrange warp) equal the oracle's (long double, Newton on P_N') as sets (R32)."""
    b = es.ref_table(d, N, "nodes1").reshape(-1, d + 1)
    _, lo = O.nodes(d, N, 1)
    key = lambda a: np.array(sorted(map(tuple, np.round(a, 12) + 0.0)))
    assert b.shape == lo.shape
    assert np.abs(key(b) - key(lo)).max() < 1e-15
    b0 = es.ref_table(d, N, "nodes0").reshape(-1, d + 1)
    assert np.abs(b0 * N - np.round(b0 * N)).max() < 1e-13
