"""The paper's robustness experiment on the GPU path (Fig. 9): the Kelvin-Helmholtz
instability on the paper's curved triangles, integrated to the paper's final time
T = 15 with the library's admissibility check on.  The entropy-stable scheme completes and its total
entropy never increases.  (The entropy-conservative run is recorded by
tools/robustness.py, not asserted: the paper reports it crashes, which is qualitative.)
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


@pytest.mark.parametrize("fm", [1, 3])
def test_khi_entropy_stable_completes(es, fm):
    import robustness as R
    summ, hist = R.run(es, I, torch, "khi", 3, 8, fm, 15.0, cfl=0.1, samples=15)
    assert summ["status"] == "completed", summ
    assert abs(summ["t_end"] - 15.0) < 1e-9
    dS = [h["dS"] for h in hist]
    assert all(b <= a + 1e-13 for a, b in zip(dS, dS[1:])), dS
    assert dS[-1] < 0.0
    assert all(h["dSdt"] <= 0.0 for h in hist[1:]), hist
