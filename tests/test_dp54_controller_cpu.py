"""Host step-size control of the Dormand-Prince 5(4) integrator (paper_2312_07874_b200.dp54_controller,
Hairer-Norsett-Wanner I, eq. II.4.13) driven by a mock step on scalar ODEs (no GPU)."""
import math

import numpy as np
import pytest

import oracle as O

es = pytest.importorskip("paper_2312_07874_b200")


class MockDP:
    """y' = f(t, y) advanced by the oracle's DP5(4) tableau, with the library's error norm"""

    def __init__(self, f, y0):
        self.c, self.A, self.b, self.bh = O.dp54_tableau()
        self.f, self.t, self.y = f, 0.0, np.array(y0, dtype=float)
        self.calls = 0

    def step(self, dt, rtol, atol):
        self.calls += 1
        k = []
        for i in range(7):
            yi = self.y + dt * sum(self.A[i, j] * k[j] for j in range(i))
            k.append(self.f(self.t + self.c[i] * dt, yi))
        y5 = self.y + dt * sum(self.b[j] * k[j] for j in range(7))
        e = dt * sum((self.b[j] - self.bh[j]) * k[j] for j in range(7))
        sc = atol + rtol * np.maximum(np.abs(self.y), np.abs(y5))
        err = math.sqrt(np.mean((e / sc) ** 2))
        if err <= 1.0:
            self.t += dt
            self.y = y5
        return err, err <= 1.0


def test_controller_reaches_T_with_tolerance():
    m = MockDP(lambda t, y: -y + np.cos(t), [1.0])
    exact = lambda t: 0.5 * (math.cos(t) + math.sin(t)) + 0.5 * math.exp(-t)  # noqa: E731
    nacc, nrej, dt = es.dp54_controller(m.step, 3.0, 1e-3, rtol=1e-8, atol=1e-10)
    assert abs(m.t - 3.0) < 1e-13
    assert abs(m.y[0] - exact(3.0)) < 1e-6
    assert nacc + nrej == m.calls and nacc > 5


def test_controller_rejects_and_recovers_from_a_large_first_step():
    m = MockDP(lambda t, y: -50.0 * (y - np.sin(t)), [0.0])
    nacc, nrej, _ = es.dp54_controller(m.step, 1.0, 0.5, rtol=1e-6, atol=1e-9)
    assert nrej >= 1 and abs(m.t - 1.0) < 1e-13


def test_controller_tolerance_controls_cost():
    counts = []
    for rtol in (1e-4, 1e-8):
        m = MockDP(lambda t, y: np.array([y[1], -y[0]]), [1.0, 0.0])
        counts.append(es.dp54_controller(m.step, 2 * math.pi, 0.1, rtol=rtol, atol=rtol * 1e-2)[0])
    # error per step ~ dt^5: steps grow like tol^(-1/5) -> 10^(4/5) = 6.3 x for 4 decades
    assert 4.0 < counts[1] / counts[0] < 9.0, counts


def test_controller_step_limit():
    m = MockDP(lambda t, y: -y, [1.0])
    with pytest.raises(es.ESError):
        es.dp54_controller(m.step, 10.0, 1e-3, rtol=1e-12, atol=1e-14, max_steps=5)


def test_controller_non_finite_error_is_a_rejection_that_shrinks_the_step():
    # a trial step that blew up reports err = nan: the controller must reject it and
    # shrink dt by facmin, not grow it by facmax
    calls = []

    def step(dt, rtol, atol):
        calls.append(dt)
        return (float("nan"), True) if dt > 0.05 else (0.5, True)

    nacc, nrej, _ = es.dp54_controller(step, 0.2, 0.1, rtol=1e-6, atol=1e-9)
    assert nrej == 1 and calls[1] == pytest.approx(0.1 * 0.2)
    assert nacc >= 1
