"""Host logic: the branch-free log / exp of the projection kernel's pointwise phases
(paper_2312_07874_b200/csrc/fastmath.cuh; PAPER App. B entropy variables) compiled
for the host with g++ and checked against numpy's long-double log / exp: at most 2 ulp."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = r'''
#include "fastmath.cuh"
extern "C" void fm_log(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = es_log_pos(x[i]); }
extern "C" void fm_exp(const double* x, double* y, long n) { for (long i = 0; i < n; ++i) y[i] = es_exp(x[i]); }
'''


@pytest.fixture(scope="module")
def fm(tmp_path_factory):
    d = tmp_path_factory.mktemp("fastmath")
    src = d / "fm.cpp"
    src.write_text(SRC)
    so = d / "fm.so"
    subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-I",
                           os.path.join(ROOT, "paper_2312_07874_b200", "csrc"), str(src), "-o", str(so)])
    return ctypes.CDLL(str(so))


def _call(f, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty_like(x)
    f(x.ctypes.data_as(ctypes.c_void_p), y.ctypes.data_as(ctypes.c_void_p), ctypes.c_long(x.size))
    return y


def _ulps(got, ref):
    ref64 = ref.astype(np.float64)
    sp = np.spacing(np.abs(ref64))
    return np.abs((got - ref).astype(np.float64)) / sp


def test_log_pos_within_2_ulp(fm):
    rng = np.random.default_rng(5)
    x = np.concatenate([np.exp(rng.uniform(-41.0, 41.0, 400_000)), rng.uniform(0.5, 2.0, 400_000),
                        1.0 + rng.uniform(-1e-6, 1e-6, 50_000),
                        [2.0, 0.5, np.sqrt(2.0), np.sqrt(0.5), np.nextafter(1.0, 2.0), np.nextafter(1.0, 0.0)]])
    got = _call(fm.fm_log, x)
    ref = np.log(x.astype(np.longdouble))
    assert _ulps(got, ref).max() <= 2.0
    assert _call(fm.fm_log, np.array([1.0]))[0] == 0.0
    # exact powers of two: k ln 2 to within an ulp
    k = np.arange(-60, 61)
    assert np.abs(_call(fm.fm_log, 2.0 ** k) - k * np.log(2.0)).max() <= 1e-14


def test_exp_within_2_ulp(fm):
    rng = np.random.default_rng(6)
    y = np.concatenate([rng.uniform(-600.0, 600.0, 400_000), rng.uniform(-1.0, 1.0, 400_000), [0.0, 1.0, -1.0]])
    got = _call(fm.fm_exp, y)
    ref = np.exp(y.astype(np.longdouble))
    assert _ulps(got, ref).max() <= 2.0
    assert _call(fm.fm_exp, np.array([0.0]))[0] == 1.0


def test_exp_log_roundtrip(fm):
    rng = np.random.default_rng(7)
    x = np.exp(rng.uniform(-30.0, 30.0, 100_000))
    back = _call(fm.fm_exp, _call(fm.fm_log, x))
    assert np.abs(back / x - 1.0).max() <= 1e-14
