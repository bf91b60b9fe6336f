"""Pins of the oracle's Newton step search (readings Q34-Q36) and of the step rules
(binary / newton / standard) — against finite differences, a brute-force root of f(alpha) = 1,
closed forms and the Theorem contract."""
import math

import numpy as np
import pytest

import graphgen as gg
import oracle as O


def _si(rng, mp, mc, eta=40.0):
    y = rng.uniform(0.0, 0.8, mp)
    z = rng.uniform(0.05, 0.9, mc)
    dy = rng.uniform(0.0, 0.02, mp)
    dz = rng.uniform(0.0, 0.03, mc)
    sP, u, SP = O.shifted_weights_packing(y, eta)
    sC, v, SC = O.shifted_weights_covering(z, eta)
    return O.SearchInputs(y, dy, z, dz, eta, sP, SP, sC, SC, u / SP, v / SC)


@pytest.mark.parametrize("seed", range(20))
def test_derivatives_match_finite_differences(seed):
    rng = np.random.default_rng(seed)
    si = _si(rng, 30, 40)
    for a in (0.5, 3.0, 17.0):
        h = 1e-6 * a
        dphi = (O.eta_phi(si, a + h) - O.eta_phi(si, a - h)) / (2 * h)
        dpsi = (O.eta_psi(si, a + h) - O.eta_psi(si, a - h)) / (2 * h)
        assert O.eta_phi_prime(si, a) == pytest.approx(dphi, rel=1e-5)
        assert O.eta_psi_prime(si, a) == pytest.approx(dpsi, rel=1e-5)


def test_singleton_derivatives_closed_form():
    si = O.SearchInputs(np.array([0.3]), np.array([0.2]), np.array([0.1]), np.array([0.4]), 7.0, 0.3, 1.0,
                        0.1, 1.0, np.array([1.0]), np.array([1.0]))
    assert O.eta_psi_prime(si, 5.0) == 7.0 * 0.2
    assert O.eta_phi_prime(si, 5.0) == 7.0 * 0.4


def _root(si, lo, hi):
    """Largest alpha with f(alpha) >= 1 by plain bisection on the monotone predicate."""
    for _ in range(200):
        mid = (lo + hi) / 2
        if O.f_at_least_one(si, mid):
            lo = mid
        else:
            hi = mid
    return lo


@pytest.mark.parametrize("seed", range(40))
def test_newton_result_is_feasible_and_eps_tight(seed):
    """The Newton answer satisfies eq:b4b_conv (f >= 1) and, when it comes from the Newton branch,
    lies within a factor (1 - eps)^2 of the largest feasible step alpha* (found by brute bisection):
    a converged iterate is eps-close to the root, and one back-off factor may follow."""
    rng = np.random.default_rng(100 + seed)
    si = _si(rng, 25, 35)
    eps = 0.1
    for a0 in (None, 2.0, 40.0):
        r = O.newton_search(si, eps, a0)
        if r.early or r.alpha < 1.0:
            continue
        assert O.f_at_least_one(si, r.alpha)
        hi = 1.0
        while O.f_at_least_one(si, hi) and hi < 1e12:
            hi *= 2
        star = _root(si, 0.0, hi)
        assert r.alpha <= star * (1 + 1e-12)
        assert r.alpha >= star * (1 - eps) ** 2 * (1 - 1e-12) or r.evals > O.NEWTON_MAX_STEPS


def test_newton_falls_back_when_f_is_constant():
    """m_P = m_C = 1 with d^(z) = d^(y): f == 1 for every alpha, so g' = 0 and Newton
    must fall back to Alg. 3 (Q35), which doubles to its evaluation cap or the early exit."""
    si = O.SearchInputs(np.array([0.5]), np.array([0.1]), np.array([0.5]), np.array([0.1]), 10.0, 0.5, 1.0,
                        0.5, 1.0, np.array([1.0]), np.array([1.0]))
    r = O.newton_search(si, 0.1, 4.0)
    b = O.binsearch(si, 0.1)
    assert r.alpha == b.alpha and r.early == b.early


def test_newton_start_without_previous_step_uses_exponential_search():
    rng = np.random.default_rng(7)
    si = _si(rng, 20, 20)
    r = O.newton_search(si, 0.1, None)
    assert O.f_at_least_one(si, r.alpha) or r.alpha < 1.0


def _nu(G, s, d):
    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg
    A = sp.csr_matrix((np.ones(len(s)), (s, d - G.n_left)), shape=(G.n_left, G.n_vertices - G.n_left))
    return int(np.sum(cg.maximum_bipartite_matching(A, perm_type="column") >= 0))


@pytest.mark.parametrize("rule", ["binary", "newton"])
def test_step_rules_solve_bipartite_matching(rule):
    """Alg. 3 and Newton both certify the LP optimum of a bipartite matching (= maximum matching,
    P:396) within (1 +- eps), scipy's Hopcroft-Karp as the reference, Theorem contract on x."""
    G = gg.bipartite_uniform(40, 50, 300, seed=3)
    s, d = G.numpy()
    r = O.solve("bmatch", s, d, G.n_vertices, eps=0.1, max_iter=5000, step_rule=rule)
    nu = _nu(G, s, d)
    assert nu / 1.1 <= r.objective <= nu * 1.1
    assert (O.incidence_M(s, d, G.n_vertices) @ r.x).max() <= 1.1 + 1e-9


def test_step_rules_iteration_counts_on_one_probe():
    """Table 3's qualitative claim on one feasible probe (M = 0.85 nu): all three
    rules reach Cx >= 1 with Px <= 1 + eps, and the searched steps (Bin, Nwt) take over ten times
    fewer MWU iterations than the standard step alpha = 1."""
    G = gg.bipartite_uniform(40, 50, 300, seed=3)
    s, d = G.numpy()
    lp = O.graph_lp("bmatch", s, d, G.n_vertices, 0.85 * _nu(G, s, d))
    its = {}
    for rule in ("standard", "binary", "newton"):
        p = O.run_probe(lp, 0.1, max_iter=200000, step_rule=rule)
        assert p.status == O.FEASIBLE, rule
        assert p.certificate() <= 1.1 + 1e-9
        its[rule] = p.t
    assert its["newton"] * 10 < its["standard"] and its["binary"] * 10 < its["standard"], its
