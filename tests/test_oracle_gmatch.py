"""Pins of the generalized-matching LP (NEXT#3) in the oracle: matrices from the
definition, feasibility verdicts against HiGHS on small instances, the Theorem contract on x."""
import numpy as np
import pytest
import scipy.optimize as so

import graphgen as gg
import oracle as O


def _highs_feasible(src, dst, nv, lb, ub):
    M = O.incidence_M(src, dst, nv).toarray()
    fin = np.isfinite(ub)
    A = np.vstack([M[fin], -M])
    b = np.concatenate([ub[fin], -lb])
    r = so.linprog(np.zeros(len(src)), A_ub=A, b_ub=b, bounds=(0, None), method="highs")
    return r.status == 0


def test_matrices_follow_the_definition():
    g = gg.complete_bipartite(2, 3)
    s, d = g.numpy()
    lb = np.array([1.0, 0.0, 0.5, 0.0, 2.0])
    ub = np.array([3.0, np.inf, 1.0, 4.0, 2.0])
    P, C = O.gmatch_matrices(s, d, 5, lb, ub)
    M = O.incidence_M(s, d, 5).toarray()
    assert np.array_equal(P.toarray(), M[[0, 2, 3, 4]] / ub[[0, 2, 3, 4]][:, None])
    assert np.array_equal(C.toarray(), M[[0, 2, 4]] / lb[[0, 2, 4]][:, None])


@pytest.mark.parametrize("seed", range(12))
def test_verdicts_match_highs(seed):
    """eps-feasibility certificates agree with exact LP feasibility where the instance is not within
    eps of the boundary (Theorem P:737-739: a feasible LP never ends INFEASIBLE; an infeasible one
    is either reported infeasible or only (1+eps)-feasible)."""
    g = gg.random_small_bipartite(6, 7, 0.5, seed=seed)
    s, d = g.numpy()
    if len(s) == 0:
        return
    rng = np.random.default_rng(seed)
    lb = np.where(rng.random(13) < 0.5, rng.uniform(0.2, 1.5, 13), 0.0)
    ub = lb + rng.uniform(0.5, 2.0, 13)
    P, C = O.gmatch_matrices(s, d, 13, lb, ub)
    if C.shape[0] == 0:
        return
    r = O.solve("mixed", P=P, C=C, eps=0.1)
    feas = _highs_feasible(s, d, 13, lb, ub)
    if feas:
        assert r.outcome == O.FEASIBLE
    if r.outcome == O.FEASIBLE:
        x = r.x
        M = O.incidence_M(s, d, 13)
        fin = np.isfinite(ub)
        assert np.all((M @ x)[fin] <= ub[fin] * 1.1 + 1e-9)
        assert np.all((M @ x) >= lb - 1e-9)


def test_app_a2_shaped_instance_is_feasible():
    g, lb, ub = gg.gmatch_instance(60, 40, seed=1)
    s, d = g.numpy()
    P, C = O.gmatch_matrices(s, d, g.n_vertices, lb.numpy(), ub.numpy())
    r = O.solve("mixed", P=P, C=C, eps=0.1)
    assert r.outcome == O.FEASIBLE
    assert r.certificate <= 1.1 + 1e-12
