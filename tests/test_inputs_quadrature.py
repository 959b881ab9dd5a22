"""The collapsed Gauss rule used for the paper's L2 error norms (degree 35): exact integration of
monomials in barycentric coordinates against the closed form a! b! c! (d!) / (a+b+c+d)! |T| (a
textbook identity, independent of the rule's construction)."""
import math

import numpy as np
import pytest

import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import quadrature as Q  # noqa: E402


@pytest.mark.parametrize("d", [2, 3])
def test_collapsed_rule_exact_to_degree_35(d):
    xi, w = Q.collapsed_gauss_rule(d, 18)
    vol = 2.0 if d == 2 else 4.0 / 3.0
    assert abs(w.sum() - vol) < 1e-14 * vol
    lam = np.concatenate([(1 + xi) / 2, 1 - ((1 + xi) / 2).sum(1, keepdims=True)], 1)  # d+1 barycentrics
    rng = np.random.default_rng(0)
    for _ in range(12):
        ex = rng.multinomial(35 if _ % 2 else int(rng.integers(1, 35)), np.ones(d + 1) / (d + 1))
        f = np.prod(lam ** ex, 1)
        exact = vol * math.factorial(d) * math.prod(math.factorial(int(k)) for k in ex) / math.factorial(int(ex.sum()) + d)
        assert abs(f @ w - exact) <= 1e-12 * exact, (ex, f @ w, exact)
