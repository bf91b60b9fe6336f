"""The oracle's own fp64 conditioning on the full-solve parity instances: the
precondition under which BASELINE's full-run tolerances can be asserted for the CUDA path."""
import pytest

import oracle as O
from instances import EPS, MAX_ITER, WELL_CONDITIONED, rounding_noise


@pytest.mark.parametrize("name", sorted(WELL_CONDITIONED))
def test_well_conditioned_full_solve(name):
    kind, mk = WELL_CONDITIONED[name]
    G = mk()
    s, d = G.numpy()
    runs = [O.solve(kind, s, d, G.n_vertices, eps=EPS[kind], max_iter=MAX_ITER, x0_scale=sc)
            for sc in (1.0, 1 + 2.0 ** -52, 1 - 2.0 ** -52)]
    for seed in (1, 2, 3):
        with rounding_noise(seed):
            runs.append(O.solve(kind, s, d, G.n_vertices, eps=EPS[kind], max_iter=MAX_ITER))
    r = runs[0]
    assert r.iters_total > 0
    for q in runs:
        assert all(p[1] != O.ITER_LIMIT for p in q.probes), [p[1] for p in q.probes]
    for q in runs[1:]:
        assert abs(q.objective - r.objective) <= 1e-6 * abs(r.objective)
        assert abs(q.bound - r.bound) <= 1e-6 * abs(r.bound)
        assert abs(q.iters_total - r.iters_total) <= 0.02 * r.iters_total
        assert [p[1] for p in q.probes] == [p[1] for p in r.probes]
