"""Measurement quadrature (error norms only; no arithmetic of the method): the collapsed-coordinate Gauss
rule of the reference simplex used for the L2 errors of the accuracy study (degree 35)."""
from __future__ import annotations

import numpy as np


def collapsed_gauss_rule(d: int, n: int):
    """Collapsed-coordinate Gauss rule on the reference simplex (vertices of P:177 / P:257) with n points
    per direction, exact for total degree 2n - 1 (n = 18: degree 35, the rule behind the paper's L2
    errors).  Gauss-Jacobi (alpha, 0) rules from scipy.special.roots_jacobi absorb the collapsed
    Jacobians (1 - eta2)/2 and (1 - eta2)(1 - eta3)^2/8.  Returns xi [n^d][d], w [n^d].  (Quadrature for
    error norms only: no arithmetic of the method.)"""
    from scipy.special import roots_jacobi
    x1, w1 = roots_jacobi(n, 0.0, 0.0)
    x2, w2 = roots_jacobi(n, 1.0, 0.0)
    if d == 2:
        e1, e2 = np.meshgrid(x1, x2, indexing="ij")
        W = np.outer(w1, w2) / 2.0
        xi = np.stack([0.5 * (1 + e1) * (1 - e2) - 1.0, e2], -1).reshape(-1, 2)
        return xi, W.reshape(-1)
    x3, w3 = roots_jacobi(n, 2.0, 0.0)
    e1, e2, e3 = np.meshgrid(x1, x2, x3, indexing="ij")
    W = w1[:, None, None] * w2[None, :, None] * w3[None, None, :] / 8.0
    xi = np.stack([0.25 * (1 + e1) * (1 - e2) * (1 - e3) - 1.0, 0.5 * (1 + e2) * (1 - e3) - 1.0, e3], -1)
    return xi.reshape(-1, 3), W.reshape(-1)
