"""Pins of the oracle's primitives against closed forms, library routines and
high-precision (mpmath) evaluations of the paper's definitions (CPU only)."""
import json
import math
import os

import mpmath
import networkx as nx
import numpy as np
import pytest
import scipy.sparse as sp

import graphgen as gg
import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
mpmath.mp.dps = 60


def mp_smax(v, eta):
    return mpmath.log(mpmath.fsum(mpmath.exp(eta * mpmath.mpf(x)) for x in v)) / eta


def mp_smin(v, eta):
    return -mpmath.log(mpmath.fsum(mpmath.exp(-eta * mpmath.mpf(x)) for x in v)) / eta


# ------------------------------------------------------------------ smax / smin
def test_smax_two_point_golden():
    ex = GOLD["smax_two_point"]
    assert O.smax(ex["v"], ex["eta"]) == pytest.approx(ex["smax"], rel=1e-15)
    assert np.allclose(O.grad_smax(ex["v"], ex["eta"]), ex["grad"], rtol=1e-15, atol=0)


def test_smax_constant_vector_golden():
    ex = GOLD["smax_constant_vector"]
    v = [ex["c"]] * ex["n"]
    assert O.smax(v, ex["eta"]) == pytest.approx(ex["smax"], rel=1e-15)
    assert O.smin(v, ex["eta"]) == pytest.approx(ex["c"] - math.log(ex["n"]) / ex["eta"], rel=1e-15)
    assert np.allclose(O.grad_smax(v, ex["eta"]), 1.0 / ex["n"], rtol=1e-15)


@pytest.mark.parametrize("seed", range(6))
def test_smax_smin_vs_mpmath_and_sandwich(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    v = rng.uniform(-2, 2, n)
    eta = float(rng.choice([0.5, 3.0, 50.0, 800.0]))
    assert O.smax(v, eta) == pytest.approx(float(mp_smax(v, eta)), rel=1e-13, abs=1e-15)
    assert O.smin(v, eta) == pytest.approx(float(mp_smin(v, eta)), rel=1e-13, abs=1e-15)
    # sandwich max <= smax <= max + ln(n)/eta ("within eps additive error")
    assert v.max() - 1e-15 <= O.smax(v, eta) <= v.max() + math.log(n) / eta + 1e-15
    assert v.min() - math.log(n) / eta - 1e-15 <= O.smin(v, eta) <= v.min() + 1e-15


@pytest.mark.parametrize("seed", range(4))
def test_gradients_are_mpmath_derivatives(seed):
    rng = np.random.default_rng(100 + seed)
    v = rng.uniform(-1, 1, 9)
    eta = 7.0
    gmax, gmin = O.grad_smax(v, eta), O.grad_smin(v, eta)
    assert abs(gmax.sum() - 1) < 1e-14 and abs(gmin.sum() - 1) < 1e-14
    for i in range(v.size):
        def fmax(t, i=i):
            w = [mpmath.mpf(x) for x in v]
            w[i] = t
            return mp_smax(w, eta)

        def fmin(t, i=i):
            w = [mpmath.mpf(x) for x in v]
            w[i] = t
            return mp_smin(w, eta)
        assert gmax[i] == pytest.approx(float(mpmath.diff(fmax, v[i])), rel=1e-12)
        assert gmin[i] == pytest.approx(float(mpmath.diff(fmin, v[i])), rel=1e-12)


def test_eta_gives_eps_over_10_smoothing():
    # eta = 10 ln(m)/eps => smax - max <= ln(m)/eta = eps/10
    for m, eps in [(2, 0.1), (1000, 0.05), (2 ** 20, 0.1)]:
        eta = O.eta_parameter(m, eps)
        assert math.log(m) / eta == pytest.approx(eps / 10, rel=1e-15)


# ------------------------------------------------------------------ init / direction
def test_init_x_golden():
    by_case = {c["case"]: c for c in GOLD["init_x"]}
    P = sp.identity(4, format="csr")
    assert np.allclose(O.init_x(P, 0.1), by_case["identity4"]["x"], rtol=1e-15)
    K3 = gg.complete_graph(3)
    M = O.incidence_M(*K3.numpy(), 3)
    x = O.init_x(M, 0.1)
    assert np.allclose(x, by_case["K3_incidence"]["x"], rtol=1e-15)
    assert (M @ x).max() == pytest.approx(by_case["K3_incidence"]["max_Px"], rel=1e-15)
    assert O.init_x(sp.csr_matrix([[2.0]]), 0.1)[0] == pytest.approx(by_case["two"]["x"][0], rel=1e-15)
    with pytest.raises(ValueError):
        O.init_x(sp.csr_matrix([[1.0, 0.0]]), 0.1)


@pytest.mark.parametrize("seed", range(5))
def test_init_x_packing_rows_at_most_eps(seed):
    lp = gg.random_planted_lp(30, 20, 10, 0.2, seed)
    P = sp.csr_matrix((lp.p_val.numpy(), lp.p_col.numpy(), lp.p_rowptr.numpy()), shape=(20, 30))
    x0 = O.init_x(P, 0.1)
    assert (P @ x0).max() <= 0.1 * (1 + 1e-12)          # S:283 post-condition


def test_direction_golden():
    for ex in GOLD["direction"]:
        sigma = O.step_sigma(ex["mode"], ex["eta"])
        d = O.direction([ex["g"]], [ex["h"]], [ex["x"]], sigma)[0]
        assert d == pytest.approx(ex["d"], rel=1e-15, abs=0), ex["cite"]
    # h = 0 convention (Q5) and g > h clipping
    assert O.direction([1.0, 2.0], [0.0, 1.0], [1.0, 1.0], 0.5).tolist() == [0.0, 0.0]


# ------------------------------------------------------------------ matrices
def _nx_graph(G):
    g = nx.Graph()
    g.add_nodes_from(range(G.n_vertices))
    s, d = G.numpy()
    g.add_edges_from(zip(s.tolist(), d.tolist()))
    return g


@pytest.mark.parametrize("G", [gg.complete_graph(5), gg.star_graph(4), gg.path_graph(6),
                               gg.random_small_graph(30, 0.2, 3), gg.random_small_bipartite(7, 9, 0.4, 1)])
def test_matrices_vs_networkx(G):
    s, d = G.numpy()
    n = G.n_vertices
    ng = _nx_graph(G)
    edgelist = list(zip(s.tolist(), d.tolist()))
    Mnx = nx.incidence_matrix(ng, nodelist=range(n), edgelist=edgelist, oriented=False)
    M = O.incidence_M(s, d, n)
    assert (M != sp.csr_matrix(Mnx)).nnz == 0
    A = nx.to_scipy_sparse_array(ng, nodelist=range(n), format="csr")
    C = O.closed_neighborhood(s, d, n)
    assert (C != sp.csr_matrix(A + sp.identity(n))).nnz == 0
    assert C.has_sorted_indices
    # O collapses to M when each (2e, 2e+1) column pair is summed; W is kron(I, [1 1])
    Op = O.pair_matrix_O(s, d, n)
    S = sp.kron(sp.identity(len(s)), np.array([[1.0], [1.0]])).tocsr()
    assert (Op @ S != M).nnz == 0
    assert (O.interweaved_W(len(s)) != S.T.tocsr()).nnz == 0
    assert np.array_equal(np.asarray(Op.sum(axis=1)).ravel(), np.array([ng.degree(v) for v in range(n)]))


def test_drop_empty_rows():
    G = gg.Graph(*[t for t in (gg.complete_graph(3).src, gg.complete_graph(3).dst)], n_vertices=5)
    M = O.incidence_M(*G.numpy(), 5)
    M2, keep = O.drop_empty_rows(M)
    assert keep.tolist() == [0, 1, 2] and M2.shape == (3, 3)


# ------------------------------------------------------------------ Phi / Psi / f
def _random_search_inputs(rng, m_p, m_c, eta, scale_dy=1.0, scale_dz=1.0):
    y = rng.uniform(0, 1, m_p)
    z = rng.uniform(0.05, 1, m_c)
    dy = rng.uniform(0, 1, m_p) * scale_dy * (rng.uniform(0, 1, m_p) < 0.8)
    dz = rng.uniform(0, 1, m_c) * scale_dz * (rng.uniform(0, 1, m_c) < 0.8)
    sP, u, SP = O.shifted_weights_packing(y, eta)
    sC, v, SC = O.shifted_weights_covering(z, eta)
    return O.SearchInputs(y, dy, z, dz, eta, sP, SP, sC, SC, u / SP, v / SC)


def _mp_psi(si, a):
    t = [mpmath.mpf(yi) + mpmath.mpf(a) * mpmath.mpf(di) for yi, di in zip(si.y, si.dy)]
    return si.eta * (mp_smax(t, si.eta) - mp_smax(si.y, si.eta))


def _mp_phi(si, a):
    t = [mpmath.mpf(zi) + mpmath.mpf(a) * mpmath.mpf(di) for zi, di in zip(si.z, si.dz)]
    return si.eta * (mp_smin(t, si.eta) - mp_smin(si.z, si.eta))


@pytest.mark.parametrize("seed", range(8))
def test_phi_psi_vs_mpmath_definition(seed):
    """Both numeric branches (Q16) agree with the P:719-720 definitions in 60-digit arithmetic."""
    rng = np.random.default_rng(seed)
    eta = float(rng.choice([20.0, 300.0, 3000.0]))
    si = _random_search_inputs(rng, int(rng.integers(2, 30)), int(rng.integers(2, 30)), eta,
                               scale_dy=float(rng.choice([1e-4, 1e-2, 1.0])),
                               scale_dz=float(rng.choice([1e-4, 1e-2, 1.0])))
    for a in [0.0, 1e-3, 0.5, 1.0, 4.0, 64.0]:
        psi, phi = O.eta_psi(si, a), O.eta_phi(si, a)
        mpsi, mphi = float(_mp_psi(si, a)), float(_mp_phi(si, a))
        # LSE branch: absolute error ~ eta * ulp(max|t|); expm1 branch: relative ~ 1e-15
        assert psi == pytest.approx(mpsi, rel=1e-11, abs=1e-12 * eta), (a, psi, mpsi)
        assert phi == pytest.approx(mphi, rel=1e-11, abs=1e-12 * eta), (a, phi, mphi)


def test_phi_psi_special_cases():
    rng = np.random.default_rng(7)
    si = _random_search_inputs(rng, 5, 6, 50.0)
    assert O.eta_psi(si, 0.0) == 0.0 and O.eta_phi(si, 0.0) == 0.0
    one = O.SearchInputs(np.array([0.3]), np.array([0.25]), np.array([0.4]), np.array([0.25]),
                         50.0, 0.3, 1.0, 0.4, 1.0, np.ones(1), np.ones(1))
    for a in [0.5, 1.0, 8.0, 1e3]:
        assert O.eta_psi(one, a) == 50.0 * a * 0.25                        # S:380 singleton
        assert O.f_at_least_one(one, a)                                     # S:390 f == 1


@pytest.mark.parametrize("seed", range(10))
def test_f_monotone_decreasing(seed):
    """Proposition Prop.MonoInc: f = Phi/Psi decreases in alpha."""
    rng = np.random.default_rng(1000 + seed)
    si = _random_search_inputs(rng, int(rng.integers(2, 50)), int(rng.integers(2, 50)), 200.0,
                               scale_dy=1e-2, scale_dz=1e-2)
    alphas = np.geomspace(1e-3, 1e3, 60)
    f = np.array([O.eta_phi(si, a) / O.eta_psi(si, a) if O.eta_psi(si, a) > 0 else np.inf for a in alphas])
    assert np.all(np.diff(f) <= 1e-9 * np.abs(f[:-1]) + 1e-12)


# ------------------------------------------------------------------ Alg. 3
def _f_ge(si, a):
    return _mp_phi(si, a) >= _mp_psi(si, a)


@pytest.mark.parametrize("seed", range(8))
def test_binsearch_brackets_true_step(seed):
    """The returned lb has f(lb) >= 1 and is within the eps bracket of the largest alpha with
    f >= 1, unless the early exit fired."""
    rng = np.random.default_rng(seed)
    eps = 0.1
    si = _random_search_inputs(rng, 12, 9, 100.0, scale_dy=1e-3, scale_dz=float(rng.choice([1e-3, 3e-2])))
    r = O.binsearch(si, eps)
    if r.alpha < 1:
        assert not _f_ge(si, 1.0)
        return
    assert _f_ge(si, r.alpha)
    if r.early:
        assert O.covering_min_after(si, r.alpha) >= 1.0
        return
    # largest alpha* with f >= 1 by mpmath bisection
    lo, hi = r.alpha, r.alpha * 4
    assert not _f_ge(si, hi) or hi > 1e12
    for _ in range(80):
        mid = (lo + hi) / 2
        lo, hi = (mid, hi) if _f_ge(si, mid) else (lo, mid)
    assert lo / (1 + eps) <= r.alpha * (1 + 1e-12) <= lo * (1 + 1e-12)


def test_binsearch_forced_branches():
    # f(1) < 1 forced: packing side grows much faster than covering side
    si = O.SearchInputs(np.array([0.5, 0.2]), np.array([1.0, 1.0]), np.array([0.3, 0.4]),
                        np.array([1e-4, 1e-4]), 100.0, 0.5, 1.0, 0.3, 1.0,
                        np.array([0.9, 0.1]), np.array([0.5, 0.5]))
    assert O.binsearch(si, 0.1).alpha < 1
    # f == 1 (singletons): doubling until min(z + a dz) >= 1; z=0.1, dz=0.1 -> a = 16
    one = O.SearchInputs(np.array([0.1]), np.array([0.1]), np.array([0.1]), np.array([0.1]),
                         50.0, 0.1, 1.0, 0.1, 1.0, np.ones(1), np.ones(1))
    r = O.binsearch(one, 0.1)
    assert r.early and r.alpha == 16.0 and r.evals == 5
    # listing stop rule (Q9) performs exactly one bisection
    rng = np.random.default_rng(3)
    si = _random_search_inputs(rng, 12, 9, 100.0, scale_dy=1e-3, scale_dz=1e-3)
    a_list = O.binsearch(si, 0.1, tol_mode="listing")
    a_pro = O.binsearch(si, 0.1, tol_mode="prose")
    assert a_list.alpha <= a_pro.alpha * (1 + 1e-15)
