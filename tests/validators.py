"""Independent exact references used to PIN the oracle (never the oracle itself):
brute-force enumeration, library LP / matching routines and closed forms.
Nothing here imports oracle/ or the product package."""
from __future__ import annotations

import itertools
from fractions import Fraction

import numpy as np
import scipy.sparse as sp
from scipy.optimize import linprog
from scipy.sparse.csgraph import maximum_bipartite_matching


def brute_max_matching(n: int, edges) -> int:
    """Largest set of pairwise vertex-disjoint edges, by exhaustive search (tiny graphs)."""
    edges = list(edges)
    best = 0

    def rec(i, used, size):
        nonlocal best
        if size + (len(edges) - i) <= best:
            return
        if i == len(edges):
            best = max(best, size)
            return
        u, v = edges[i]
        if u not in used and v not in used:
            rec(i + 1, used | {u, v}, size + 1)
        rec(i + 1, used, size)

    rec(0, frozenset(), 0)
    return best


def scipy_bipartite_matching(n_left: int, n_right: int, src, dst) -> int:
    """scipy.sparse.csgraph.maximum_bipartite_matching (compiled Hopcroft-Karp)."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64) - n_left
    B = sp.csr_matrix((np.ones(src.size), (src, dst)), shape=(n_left, n_right))
    return int((maximum_bipartite_matching(B, perm_type="column") >= 0).sum())


def half_integral_vcover(n: int, edges) -> Fraction:
    """Fractional vertex cover optimum by enumeration over {0, 1/2, 1}^n (the vertex-cover LP
    is half-integral); exact rationals."""
    best = None
    vals = (Fraction(0), Fraction(1, 2), Fraction(1))
    for x in itertools.product(vals, repeat=n):
        if all(x[u] + x[v] >= 1 for u, v in edges):
            s = sum(x)
            if best is None or s < best:
                best = s
    return best


def brute_densest(n: int, edges) -> Fraction:
    """max over non-empty S of |E(S)|/|S| by enumerating all subsets (n <= 14)."""
    best = Fraction(0)
    for mask in range(1, 1 << n):
        k = bin(mask).count("1")
        e = sum(1 for u, v in edges if (mask >> u) & 1 and (mask >> v) & 1)
        best = max(best, Fraction(e, k))
    return best


def highs_lp(c, A_ub=None, b_ub=None, maximize=False) -> float:
    """scipy.optimize.linprog (HiGHS) optimum of  min/max c^T x  s.t. A_ub x <= b_ub, x >= 0."""
    c = np.asarray(c, dtype=float)
    res = linprog(-c if maximize else c, A_ub=A_ub, b_ub=b_ub, bounds=(0, None), method="highs")
    assert res.status == 0, res.message
    return -res.fun if maximize else res.fun


def highs_matching(n: int, edges) -> float:
    m = len(edges)
    A = np.zeros((n, m))
    for e, (u, v) in enumerate(edges):
        A[u, e] = A[v, e] = 1
    return highs_lp(np.ones(m), A, np.ones(n), maximize=True)


def highs_vcover(n: int, edges) -> float:
    A = np.zeros((len(edges), n))
    for e, (u, v) in enumerate(edges):
        A[e, u] = A[e, v] = 1
    return highs_lp(np.ones(n), -A, -np.ones(len(edges)))


def highs_domset(n: int, edges) -> float:
    A = np.eye(n)
    for u, v in edges:
        A[u, v] = A[v, u] = 1
    return highs_lp(np.ones(n), -A, -np.ones(n))


def highs_densest_primal(n: int, edges) -> float:
    """Charikar's LP (eq:densetSubgraphLP form): max sum x_e s.t. x_e <= y_u, x_e <= y_v,
    sum y <= 1 — a library LP solve independent of the dual the solver uses."""
    m = len(edges)
    rows = []
    for e, (u, v) in enumerate(edges):
        for w in (u, v):
            r = np.zeros(m + n)
            r[e] = 1
            r[m + w] = -1
            rows.append(r)
    r = np.zeros(m + n)
    r[m:] = 1
    rows.append(r)
    b = np.zeros(len(rows))
    b[-1] = 1
    c = np.concatenate([np.ones(m), np.zeros(n)])
    return highs_lp(c, np.array(rows), b, maximize=True)
