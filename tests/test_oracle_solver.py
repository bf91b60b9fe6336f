"""Pins of the oracle's Alg. 2 probe and outer searches: forced instances, the Theorem's
contract, invariants, and LP optima from brute force,
closed forms and library solvers (HiGHS, Hopcroft-Karp)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp

import graphgen as gg
import oracle as O
import validators as V

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def _csr(lp_p):
    rp, c, v = lp_p
    return sp.csr_matrix((v.numpy(), c.numpy(), rp.numpy()), shape=(rp.numel() - 1, int(c.max()) + 1 if c.numel() else 0))


def _lp_mats(lp):
    P = sp.csr_matrix((lp.p_val.numpy(), lp.p_col.numpy(), lp.p_rowptr.numpy()),
                      shape=(lp.p_rowptr.numel() - 1, lp.n))
    C = sp.csr_matrix((lp.c_val.numpy(), lp.c_col.numpy(), lp.c_rowptr.numpy()),
                      shape=(lp.c_rowptr.numel() - 1, lp.n))
    return P, C


# ------------------------------------------------------------------ forced instances
def test_forced_infeasible_and_feasible_scalars():
    p = O.run_probe(O.mixed_lp(sp.csr_matrix([[2.0]]), sp.csr_matrix([[1.0]])), 0.1)
    assert p.status == O.INFEASIBLE
    # P = C = [[1]] is feasible only at the tight point x = 1; the literal direction rule
    # gives g = h, hence d = 0 and INFEASIBLE — the paper's algorithm, not
    # SPEC S:305's expectation (reading Q34)
    p = O.run_probe(O.mixed_lp(sp.csr_matrix([[1.0]]), sp.csr_matrix([[1.0]])), 0.1)
    assert p.status == O.INFEASIBLE and p.reason == "MAXD_ZERO"
    # x in [1/2, 1] feasible: found, with x_out = 1/2 (min Cx = 1) and rho = 1/2
    p = O.run_probe(O.mixed_lp(sp.csr_matrix([[1.0]]), sp.csr_matrix([[2.0]])), 0.1)
    assert p.status == O.FEASIBLE
    assert 0.5 <= p.x[0] and p.x_out()[0] == 0.5 and p.certificate() <= 1.1


def test_infeasible_by_construction():
    P, C = _lp_mats(gg.infeasible_lp(6, 0))
    assert O.run_probe(O.mixed_lp(P, C), 0.1).status == O.INFEASIBLE


def test_empty_covering_row_is_infeasible():
    P = sp.csr_matrix(np.eye(2))
    C = sp.csr_matrix(np.array([[1.0, 1.0], [0.0, 0.0]]))
    p = O.Probe(O.mixed_lp(P, C), 0.1)
    assert p.status == O.INFEASIBLE and p.reason == "EMPTY_COVER_ROW"


# ------------------------------------------------------------------ Theorem contract + invariants
@pytest.mark.parametrize("seed", range(12))
def test_planted_feasible_contract_and_invariants(seed):
    """Feasible-by-design instances are never reported INFEASIBLE; x_out has
    min Cx = 1 and max Px <= 1 + eps*(1+0.2) (reading Q6 bound); potential
    non-increasing, x monotone, cached y,z drift <= 1e-9."""
    eps = 0.1
    lp = gg.random_planted_lp(int(10 + seed), 8, 6, 0.3, seed)
    P, C = _lp_mats(lp)
    p = O.Probe(O.mixed_lp(P, C), eps, max_iter=3000)
    pot_prev = O.smax(p.y, p.eta) - O.smin(p.z, p.eta)
    x_prev = p.x.copy()
    while p.step() == O.RUNNING:
        pot = O.smax(p.y, p.eta) - O.smin(p.z, p.eta)
        assert pot <= pot_prev + 1e-9
        assert np.all(p.x >= x_prev)
        assert np.max(np.abs(p.y - p.lp.P @ p.x)) <= 1e-9 * max(1.0, np.abs(p.y).max())
        assert np.max(np.abs(p.z - p.lp.C @ p.x)) <= 1e-9 * max(1.0, np.abs(p.z).max())
        pot_prev, x_prev = pot, p.x.copy()
    assert p.status == O.FEASIBLE, (p.status, p.reason, p.t)
    xo = p.x_out()
    assert (C @ xo).min() >= 1 - 1e-12
    assert (P @ xo).max() <= 1 + 1.2 * eps


# ------------------------------------------------------------------ optima of the §3 LPs
def _graphs_for(kind):
    fam = {
        "K3,3": gg.complete_bipartite(3, 3), "K3": gg.complete_graph(3), "P3": gg.path_graph(3),
        "K5": gg.complete_graph(5), "S4": gg.star_graph(4), "K6": gg.complete_graph(6),
    }
    return fam


@pytest.mark.parametrize("ex", GOLD["lp_optima"], ids=lambda e: f'{e["kind"]}-{e["graph"]}')
def test_golden_lp_optima(ex):
    G = _graphs_for(ex["kind"])[ex["graph"]]
    s, d = G.numpy()
    eps = 0.1
    r = O.solve(ex["kind"], s, d, G.n_vertices, eps=eps)
    opt = ex["opt"]
    _check_objective(ex["kind"], r, opt, eps)


def _check_objective(kind, r, opt, eps):
    """Objective within the (1 +- eps) band the Theorem gives (P:737-739 with the outer
    eps/4 bracket, Q14); one-sided exact bounds where x_out is exactly feasible."""
    obj = r.objective
    if kind in ("bmatch", "match", "packing"):
        # x_out / rho is feasible => obj / rho <= opt; probes below opt succeed => obj >= opt/(1+eps)
        assert obj <= r.certificate * opt * (1 + 1e-9) if not math.isnan(r.certificate) else obj <= opt * (1 + 1e-9)
        assert obj >= opt / (1 + eps) * (1 - 1e-9)
    elif kind in ("vcover", "domset", "covering"):
        assert obj >= opt * (1 - 1e-9)                  # C x_out >= 1 is exact (Q15)
        assert obj <= opt * (1 + 1.2 * eps)
    else:  # densest: D within (1+eps) of the max density
        assert opt * (1 - 1e-9) / (1 + 0.2 * eps) <= obj <= opt * (1 + eps) * (1 + 1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_bmatch_vs_matching_references(seed):
    G = gg.random_small_bipartite(6, 7, 0.35, seed)
    s, d = G.numpy()
    edges = list(zip(s.tolist(), d.tolist()))
    opt = V.brute_max_matching(G.n_vertices, edges)
    assert opt == V.scipy_bipartite_matching(6, 7, s, d)
    assert opt == pytest.approx(V.highs_matching(G.n_vertices, edges))     # no integrality gap P:396
    _check_objective("bmatch", O.solve("bmatch", s, d, G.n_vertices, eps=0.1), opt, 0.1)


@pytest.mark.parametrize("n", [2, 4, 7])
def test_bmatch_complete_bipartite_closed_form(n):
    G = gg.complete_bipartite(n, n)
    r = O.solve("bmatch", *G.numpy(), G.n_vertices, eps=0.1)
    _check_objective("bmatch", r, n, 0.1)


@pytest.mark.parametrize("seed", range(5))
def test_vcover_vs_enumeration_and_highs(seed):
    G = gg.random_small_graph(9, 0.35, seed)
    s, d = G.numpy()
    if len(s) == 0:
        pytest.skip("empty")
    edges = list(zip(s.tolist(), d.tolist()))
    opt = float(V.half_integral_vcover(G.n_vertices, edges))
    assert opt == pytest.approx(V.highs_vcover(G.n_vertices, edges))
    _check_objective("vcover", O.solve("vcover", s, d, G.n_vertices, eps=0.1), opt, 0.1)


@pytest.mark.parametrize("nk", [(10, 3), (12, 4)])
def test_vcover_regular_closed_form(nk):
    n, k = nk
    G = gg.circulant_regular(n, k)
    _check_objective("vcover", O.solve("vcover", *G.numpy(), n, eps=0.1), n / 2, 0.1)


@pytest.mark.parametrize("nk", [(10, 3), (12, 4), (12, 5)])
def test_domset_regular_closed_form_and_highs(nk):
    n, k = nk
    G = gg.circulant_regular(n, k)
    s, d = G.numpy()
    edges = list(zip(s.tolist(), d.tolist()))
    assert V.highs_domset(n, edges) == pytest.approx(n / (k + 1))
    _check_objective("domset", O.solve("domset", s, d, n, eps=0.1), n / (k + 1), 0.1)


@pytest.mark.parametrize("seed", range(4))
def test_domset_vs_highs(seed):
    G = gg.random_small_graph(14, 0.2, 10 + seed)
    s, d = G.numpy()
    opt = V.highs_domset(G.n_vertices, list(zip(s.tolist(), d.tolist())))
    _check_objective("domset", O.solve("domset", s, d, G.n_vertices, eps=0.05), opt, 0.05)


@pytest.mark.parametrize("seed", range(5))
def test_densest_vs_brute_force_and_highs(seed):
    G = gg.random_small_graph(10, 0.4, 20 + seed)
    s, d = G.numpy()
    if len(s) == 0:
        pytest.skip("empty")
    edges = list(zip(s.tolist(), d.tolist()))
    opt = float(V.brute_densest(G.n_vertices, edges))
    assert opt == pytest.approx(V.highs_densest_primal(G.n_vertices, edges))  # Charikar duality
    _check_objective("densest", O.solve("densest", s, d, G.n_vertices, eps=0.1), opt, 0.1)


@pytest.mark.parametrize("nk", [(8, 3), (10, 4)])
def test_densest_regular_closed_form(nk):
    n, k = nk
    G = gg.circulant_regular(n, k)
    _check_objective("densest", O.solve("densest", *G.numpy(), n, eps=0.1), k / 2, 0.1)


@pytest.mark.slow
def test_c1_full_size_vs_hopcroft_karp():
    """BJ:7: the exact maximum matching of c1 (scipy Hopcroft-Karp) checks the objective."""
    G = gg.config_graph("c1")
    s, d = G.numpy()
    opt = V.scipy_bipartite_matching(1000, 1000, s, d)
    r = O.solve("bmatch", s, d, G.n_vertices, eps=0.1)
    _check_objective("bmatch", r, opt, 0.1)


def test_step_counts_standard_vs_search():
    """Qualitative Table 3 claim: step-size search needs far fewer MWU iterations
    than the standard step alpha = 1 on the same probe."""
    G = gg.random_small_bipartite(20, 20, 0.2, 5)
    s, d = G.numpy()
    lp = O.graph_lp("bmatch", s, d, G.n_vertices, 5.0)
    p_bin = O.run_probe(lp, 0.1, max_iter=20000)
    p_std = O.Probe(lp, 0.1, max_iter=20000)
    while p_std.step(alpha=1.0) == O.RUNNING:
        pass
    assert p_bin.status == p_std.status == O.FEASIBLE
    assert p_bin.t * 10 < p_std.t


def test_iter_limit_counts_as_infeasible_in_the_outer_search():
    """Q14: a probe that reaches max_iter is ITER_LIMIT (Alg. 2's loop run for at
    most max_iter iterations), and the outer geometric bisection treats it as
    infeasible: the packing search (maximise) then lowers its upper end, the covering
    search (minimise) raises its lower end.  With max_iter = 1 most probes cannot finish; the
    recorded probe sequence is replayed against the bisection rule with ITER_LIMIT as infeasible,
    and the returned witnesses still satisfy the LP."""
    G = gg.erdos_renyi(60, 240, seed=3)
    s, d = G.numpy()
    P = O.incidence_M(s, d, G.n_vertices)
    L, H, _ = O.packing_bracket(P, 0.1)
    p = O.run_probe(O.packing_lp(P, math.sqrt(L * H)), 0.1, max_iter=1)
    assert p.status == O.ITER_LIMIT and p.t == 1
    C = P.T.tocsr()
    Lc, Hc, _ = O.covering_bracket(C)
    for kind, eps, lo, hi, sense in (("match", 0.1, L, H, +1), ("vcover", 0.05, Lc, Hc, -1)):
        r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=1)
        assert any(q[1] == O.ITER_LIMIT for q in r.probes)
        for B, status, t, _ in r.probes:
            assert B == math.sqrt(lo * hi) and t <= 1
            ok = status == O.FEASIBLE                        # ITER_LIMIT: not ok (infeasible)
            if (ok and sense > 0) or (not ok and sense < 0):
                lo = B
            else:
                hi = B
        assert r.bound == (lo if sense > 0 else hi)
        if sense > 0:                                        # Theorem P:737-739: P x <= (1 + eps)
            assert (P @ r.x).max() <= 1 + eps + 1e-12
        else:
            assert (C @ r.x).min() >= 1 - 1e-12
