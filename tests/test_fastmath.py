"""The kernels' fp64 exp / expm1 (paper_2307_03307_b200/csrc/fastmath.cuh, one reduction and one
polynomial for both) against 50-digit mpmath: within 4 ulps over the arguments the hot loops see
(covering side x <= 0 down to underflow, packing side x >= 0, the step search's tiny arguments),
and subnormal exp within 1e-310 absolute (the weight-parity floor)."""
import ctypes
import os
import subprocess

import mpmath
import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fm(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("fm") / "fm.so")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                    os.path.join(ROOT, "tests", "native", "fastmath_host.cpp")], check=True)
    L = ctypes.CDLL(so)
    L.fm_eval.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long]

    def ev(x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        em, q = np.empty_like(x), np.empty_like(x)
        L.fm_eval(x.ctypes.data, em.ctypes.data, q.ctypes.data, x.size)
        return em, q
    return ev


def _ulps(a, b):
    return abs(a - b) / max(np.spacing(abs(b)), 5e-324)


def test_exp_expm1_accuracy(fm):
    mpmath.mp.dps = 50
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.uniform(-745, 0, 1500), rng.uniform(0, 709, 500), rng.uniform(-1, 1, 800),
                         rng.uniform(-1e-6, 1e-6, 300), -np.logspace(-300, 2.8, 300), np.logspace(-300, 2.8, 300),
                         [0.0, -0.0, 1e-320, -0.34657359, 0.34657359, -0.6931471805599453, 709.7]])
    em, q = fm(xs)
    worst_q = worst_em = 0.0
    for x, a, b in zip(xs, em, q):
        eq = float(mpmath.exp(mpmath.mpf(x)))
        eem = float(mpmath.expm1(mpmath.mpf(x)))
        if eq >= 2.2250738585072014e-308:
            worst_q = max(worst_q, _ulps(b, eq))
        else:
            assert abs(b - eq) <= 1e-310, (x, b, eq)
        worst_em = max(worst_em, _ulps(a, eem))
    assert worst_q <= 4 and worst_em <= 4, (worst_q, worst_em)


def test_table_exp_accuracy(tmp_path):
    so = str(tmp_path / "fm2.so")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                    os.path.join(ROOT, "tests", "native", "fastmath_host.cpp")], check=True)
    L = ctypes.CDLL(so)
    L.fm_exp_tab.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
    mpmath.mp.dps = 50
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(-745, 0, 3000), rng.uniform(-2, 2, 2000), rng.uniform(0, 709, 500),
                         [0.0, -1e-300, 1e-12, -0.0013538, 709.7, -745.1]])
    q = np.empty_like(xs)
    L.fm_exp_tab(xs.ctypes.data, q.ctypes.data, xs.size)
    worst = 0.0
    for x, b in zip(xs, q):
        e = float(mpmath.exp(mpmath.mpf(x)))
        if e >= 2.2250738585072014e-308:
            worst = max(worst, _ulps(b, e))
        else:
            assert abs(b - e) <= 1e-310, (x, b, e)
    assert worst <= 2, worst


def test_table_expm1_exp_accuracy(tmp_path):
    so = str(tmp_path / "fm3.so")
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", so,
                    os.path.join(ROOT, "tests", "native", "fastmath_host.cpp")], check=True)
    L = ctypes.CDLL(so)
    L.fm_expm1_exp_tab.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_long]
    mpmath.mp.dps = 50
    rng = np.random.default_rng(12)
    xs = np.concatenate([rng.uniform(-745, 0, 2000), rng.uniform(-1, 1, 2000), rng.uniform(-0.02, 0.02, 2000),
                         rng.uniform(-1e-5, 1e-5, 500), rng.uniform(0, 700, 500), -np.logspace(-300, 2.8, 300),
                         np.logspace(-300, 2.8, 300), [0.0, 0.0027076, -0.0027076, 0.00135, -0.00135]])
    em, q = np.empty_like(xs), np.empty_like(xs)
    L.fm_expm1_exp_tab(xs.ctypes.data, em.ctypes.data, q.ctypes.data, xs.size)
    wq = we = 0.0
    for x, a, b in zip(xs, em, q):
        eq = float(mpmath.exp(mpmath.mpf(x)))
        eem = float(mpmath.expm1(mpmath.mpf(x)))
        if eq >= 2.2250738585072014e-308:
            wq = max(wq, _ulps(b, eq))
        else:
            assert abs(b - eq) <= 1e-310, (x, b, eq)
        we = max(we, _ulps(a, eem))
    assert wq <= 3 and we <= 4, (wq, we)


def test_special_arguments(fm):
    em, q = fm([-np.inf, -800.0, 710.0, 0.0])
    assert q[0] == 0.0 and em[0] == -1.0 and q[1] == 0.0
    assert np.isinf(q[2]) and em[3] == 0.0 and q[3] == 1.0
