"""Butcher tableaux passed to es_step_erk (test / experiment tooling, not product code).

dop853(): the 12-stage 8th-order Dormand-Prince method (Hairer, Norsett & Wanner I, II.5; the paper's
integrator), read from scipy's published coefficient table (scipy.integrate._ivp.
dop853_coefficients) -- not typed from memory.  rk4(): the classical four-stage method (R17)."""
from __future__ import annotations

import numpy as np


def dop853():
    from scipy.integrate._ivp import dop853_coefficients as D
    s = D.N_STAGES
    return np.array(D.A[:s, :s], dtype=np.float64), np.array(D.B, dtype=np.float64), np.array(D.C[:s], dtype=np.float64)


def rk4():
    A = np.zeros((4, 4))
    A[1, 0], A[2, 1], A[3, 2] = 0.5, 0.5, 1.0
    return A, np.array([1.0, 2.0, 2.0, 1.0]) / 6.0, np.array([0.0, 0.5, 0.5, 1.0])


def erk_step(f, t, y, dt, A, b, c):
    """one explicit Runge-Kutta step (reference loop for tests)"""
    k = []
    for i in range(len(b)):
        yi = y + dt * sum(A[i, j] * k[j] for j in range(i) if A[i, j] != 0.0) if i else y
        k.append(f(t + c[i] * dt, yi))
    return y + dt * sum(b[j] * k[j] for j in range(len(b)) if b[j] != 0.0)
