"""The Dormand-Prince 8 tableau handed to es_step_erk (the paper's integrator): row sums equal
the nodes, sum b = 1, and the method converges at order 8 on a nonlinear ODE with a closed-form
solution (y' = y^2, y(0) = 1/2: y = 1/(2 - t)) -- a plausible transcription slip fails the order."""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import tableaux as T  # noqa: E402


def _err(A, b, c, n):
    y, t, dt = np.array([0.5]), 0.0, 1.0 / n
    for _ in range(n):
        y = T.erk_step(lambda t, y: y * y, t, y, dt, A, b, c)
        t += dt
    return abs(y[0] - 1.0 / (2.0 - 1.0))


def test_dop853_consistency_and_order_8():
    A, b, c = T.dop853()
    assert A.shape == (12, 12) and np.abs(np.triu(A)).max() == 0.0
    assert np.abs(A.sum(1) - c).max() < 1e-14 and abs(b.sum() - 1.0) < 1e-14
    e1, e2 = _err(A, b, c, 8), _err(A, b, c, 16)
    assert 7.5 < math.log2(e1 / e2) < 8.6, (e1, e2)


def test_rk4_order_4():
    A, b, c = T.rk4()
    e1, e2 = _err(A, b, c, 16), _err(A, b, c, 32)
    assert 3.8 < math.log2(e1 / e2) < 4.2
