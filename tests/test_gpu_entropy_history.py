"""Entropy history on the GPU path: Taylor-Green vortex on curved tets, RK4.
EC interface flux: the semi-discrete entropy rate vanishes to roundoff at every sampled state and
the total entropy changes only by the (small) RK4 time-integration error; ES: the rate is negative
and the total entropy decreases monotonically.  Conserved totals drift only at roundoff.
"""
import os
import sys

import pytest

import es_inputs as I

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.fixture(scope="module")
def es():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_07874_b200 as es
    return es


def test_tgv_entropy_history(es):
    import entropy_history as H
    ec, _ = H.run(es, I, torch, 3, 3, 0.3, 60, 20, 0, warp="paper")
    esh, _ = H.run(es, I, torch, 3, 3, 0.3, 60, 20, 1, warp="paper")
    ejh, _ = H.run(es, I, torch, 3, 3, 0.3, 60, 20, 2, warp="paper")  # entropy-jump dissipation (R27)
    mdh, _ = H.run(es, I, torch, 3, 3, 0.3, 60, 20, 3, warp="paper")  # matrix dissipation (R28)
    for hist in (ejh, mdh):
        for h in hist:
            assert h["dSdt"] < 0.0, h
        S = [h["S"] for h in hist]
        assert all(b < a for a, b in zip(S, S[1:])), S
    for h in ec:
        assert abs(h["dSdt"]) <= 1e-12 * h["dSdt_scale"], h
    for h in esh:
        assert h["dSdt"] < 0.0, h
    S_es = [h["S"] for h in esh]
    assert all(b < a for a, b in zip(S_es, S_es[1:])), S_es
    S_ec = [h["S"] for h in ec]
    assert abs(S_ec[-1] - S_ec[0]) < 1e-3 * abs(S_es[-1] - S_es[0]) + 1e-12 * abs(S_ec[0]), (S_ec, S_es)
    for hist in (ec, esh, ejh, mdh):
        t0 = hist[0]["totals"]
        for h in hist[1:]:
            for a, b in zip(t0, h["totals"]):
                assert abs(b - a) <= 1e-11 * max(1.0, abs(a)), (t0, h["totals"])
