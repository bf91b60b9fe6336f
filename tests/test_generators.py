"""Seeded input generators (graphgen/, shared by oracle and CUDA path, no MWU arithmetic)."""
import itertools
import math

import numpy as np

import graphgen as gg


def test_rgg_matches_brute_force():
    g = gg.rgg(8, avg_degree=10.0, seed=3)
    rng = np.random.default_rng(3)
    pts = rng.random((256, 2))
    r = math.sqrt(10.0 / (math.pi * 256))
    ref = {(i, j) for i, j in itertools.combinations(range(256), 2) if ((pts[i] - pts[j]) ** 2).sum() < r * r}
    s, d = g.numpy()
    assert (s < d).all()
    assert set(zip(s.tolist(), d.tolist())) == ref


def test_biadjacency_doubles_the_edges():
    g = gg.cycle_graph(7)
    b = gg.biadjacency(g)
    s, d = b.numpy()
    assert b.n_left == 7 and b.n_vertices == 14 and b.n_edges == 14
    assert (s < 7).all() and (d >= 7).all()
    assert len(set(zip(s.tolist(), d.tolist()))) == 14


def test_disjoint_union_and_perturbed_copies():
    u = gg.disjoint_union(gg.star_graph(3), gg.complete_bipartite(2, 2))
    s, d = u.numpy()
    assert u.n_vertices == 8 and u.n_edges == 7 and s[3:].min() >= 4
    q = gg.plus_random_edges(gg.complete_bipartite(3, 4), 2, seed=1)
    assert q.n_edges == 14
