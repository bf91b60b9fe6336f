"""Parity at BASELINE scale (SURVEY §4 T3/T4, §8(d) "reduced"): the BASELINE graphs themselves (c2,
c3 at full size) and same-recipe reduced instances of c4 (R-MAT scale 18 / 20) and c5 (2^18+2^18,
2^20+2^20), in the bench's launch configuration, 50 iterations in lockstep with the oracle on the
same seeded graph:
  - standard steps (alpha = 1): every vector within 1e-10 relative (x, y, z, weights,
    g, h) and d, d^(y), d^(z) within 1e-10 plus the 1 - g/h cancellation allowance;
  - searched steps (Alg. 3 on both sides): the same vectors within max(1e-10, 10 x the oracle's own
    rounding-noise drift), identical step sizes;
  - the L2-blocked multi-block edge order (small block_l / block_r) under the same checks;
and full solves on reduced instances (chaotic: printed spread, Theorem contract asserted)."""
import math

import numpy as np
import pytest

import graphgen as gg
import oracle as O
from gpu_common import lockstep, self_drift, solver_for
from instances import EPS

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
KIND = {"c1": "bmatch", "c2": "vcover", "c3": "domset", "c4": "densest", "c5": "bmatch"}


def _instance(cfg, sd):
    G = gg.config_graph(cfg, scale_down=sd, seed=1, device="cuda")
    return G, G.numpy()


def _bound(kind, G, s, d, eps):
    """A bound just above the optimum (the oracle's probes there take the longest): the first
    outer-bisection bound of the solve's bracket, halved towards the lower end twice."""
    deg = np.bincount(np.concatenate([s, d]).astype(np.int64), minlength=G.n_vertices)
    E, npr, D = len(s), int(np.count_nonzero(deg)), int(deg.max())
    if kind == "densest":
        L, H = E / npr, D / 2.0
    elif kind == "bmatch":
        L, H = E / D, float(E)
    elif kind == "vcover":
        L, H = E / D, float(npr)
    else:
        L, H = G.n_vertices / (D + 1), float(G.n_vertices)
    return math.sqrt(L * H)


@pytest.mark.parametrize("cfg,sd,phase", [("c2", 0, True), ("c3", 0, False), ("c4", 6, True), ("c4", 4, False),
                                          ("c5", 8, True), ("c5", 6, False)])
def test_standard_step_lockstep_at_scale(cuda_ok, cfg, sd, phase):
    kind = KIND[cfg]
    G, (s, d) = _instance(cfg, sd)
    B = _bound(kind, G, s, d, EPS[kind])
    probe = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), EPS[kind], max_iter=5000)
    S = solver_for(kind, G)
    recs = lockstep(S, probe, B, EPS[kind], 50, alphas=[1.0] * 50, strict_derived=True, phase_check=phase)
    print(f"{cfg}/2^{sd}: {len(recs) - 1} iterations, max x err {max(r['x'] for r in recs):.2e}")


@pytest.mark.parametrize("cfg,sd", [("c4", 6), ("c5", 8)])
def test_searched_lockstep_at_scale(cuda_ok, cfg, sd):
    kind = KIND[cfg]
    G, (s, d) = _instance(cfg, sd)
    B = _bound(kind, G, s, d, EPS[kind])
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    probe = O.Probe(lp, EPS[kind], max_iter=5000)
    S = solver_for(kind, G)
    recs = lockstep(S, probe, B, EPS[kind], 50, alphas=None, drift=self_drift(lp, EPS[kind], None, 50))
    print(f"{cfg}/2^{sd} searched: {len(recs) - 1} iterations compared")


@pytest.mark.parametrize("cfg,sd,bl,br", [("c4", 8, 12, 10), ("c5", 10, 13, 11)])
def test_multiblock_order_lockstep(cuda_ok, cfg, sd, bl, br):
    """Reduced instances with row blocks of 2^bl x 2^br so the L2-blocked internal edge order has
    tens of (source, destination) block pairs, as c4 / c5 have at full size."""
    kind = KIND[cfg]
    G, (s, d) = _instance(cfg, sd)
    B = _bound(kind, G, s, d, EPS[kind])
    probe = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), EPS[kind], max_iter=5000)
    S = solver_for(kind, G, block_l=bl, block_r=br)
    lockstep(S, probe, B, EPS[kind], 50, alphas=[1.0] * 50, strict_derived=True)


@pytest.mark.parametrize("cfg,sd", [("c4", 12), ("c5", 15), ("c2", 9), ("c3", 11)])
def test_reduced_full_solve(cuda_ok, cfg, sd):
    """Full solve (max_iter 5000) on a same-recipe reduced instance: random graphs are chaotic in
    fp64, so the objective / iteration spread against the oracle is printed and the
    asserted contract is the Theorem's on the GPU's x plus both being (1+eps)-approximate
    answers of the same LP (objectives within 2 eps)."""
    kind = KIND[cfg]
    eps = EPS[kind]
    G, (s, d) = _instance(cfg, sd)
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=5000)
    S = solver_for(kind, G)
    assert S.solve(eps, 5000) == "feasible"
    st = S.stats()
    print(f"{cfg}/2^{sd}: objective {st['objective']:.9g} vs oracle {r.objective:.9g} "
          f"(rel {abs(st['objective'] - r.objective) / r.objective:.2e}); iterations {st['iters_total']} vs "
          f"{r.iters_total}; probes {st['probes']} vs {len(r.probes)}; near ties {st['near_tie_count']}")
    assert abs(st["objective"] - r.objective) <= 2 * eps * abs(r.objective)
    x = S.x().cpu().numpy()
    lp = O.graph_lp(kind, s, d, G.n_vertices, st["bound"])
    assert (lp.C @ x).min() >= 1 - 1e-9
    if not math.isnan(st["certificate"]):
        assert (lp.P @ x).max() == pytest.approx(st["certificate"], rel=1e-9)
