"""The Newton step search and the standard step (Alg. 1) on the
GPU against the oracle: every accepted step size equals the oracle's Newton search replayed on the
GPU's own cached vectors (warm-started from the GPU's previous step, readings Q34-Q36), and full
solves certify the Theorem contract with the oracle's objective."""
import math

import numpy as np
import pytest

import graphgen as gg
import oracle as O
from gpu_common import Gpu, solver_for
from instances import EPS, MAX_ITER, WELL_CONDITIONED

pytestmark = pytest.mark.gpu

GRAPHS = {"bmatch": gg.bipartite_uniform(200, 300, 5000, seed=3), "match": gg.rmat(10, 8, seed=4),
          "vcover": gg.erdos_renyi(2000, 16000, seed=5), "domset": gg.rmat(11, 16, seed=6),
          "densest": gg.rmat(10, 16, seed=7)}


@pytest.mark.parametrize("kind", sorted(GRAPHS))
def test_newton_step_parity(cuda_ok, kind):
    G = GRAPHS[kind]
    s, d = G.numpy()
    eps = EPS[kind]
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=300)
    B = [p[0] for p in r.probes if p[1] == O.FEASIBLE][-1]
    S = solver_for(kind, G, step_rule="newton")
    S.set_record(True)
    S.probe_begin(B, eps)
    gpu = Gpu(S)
    prev, n = None, 0
    for t in range(40):
        before = gpu.state()
        st = S.step(0.0)
        ph = gpu.phase()
        sc = before["sc"]
        si = O.SearchInputs(before["y"], ph["dy"], before["z"], ph["dz"], sc["eta"], sc["sP"], sc["SP"], sc["sC"],
                            sc["SC"], before["wp"], before["wc"])
        ref = O.newton_search(si, eps, prev)
        assert ph["alpha"] == pytest.approx(ref.alpha, rel=1e-9), (t, ph["alpha"], ref.alpha)
        n += 1
        if st != "running":
            break
        prev = ph["alpha"]
    assert n >= 3


def test_standard_step_is_alpha_one(cuda_ok):
    G = GRAPHS["bmatch"]
    S = solver_for("bmatch", G, step_rule="standard")
    S.probe_begin(200.0, 0.1)
    for _ in range(5):
        assert S.step(0.0) == "running"
        assert S.scalars()["alpha_last"] == 1.0


@pytest.mark.parametrize("name", ["bmatch-bu21", "match-er21", "domset-K25,26", "densest-bu310"])
def test_newton_full_solve(cuda_ok, name):
    """Full solve with Newton steps: same optimum as the oracle's Newton solve (1e-6 on these
    well-conditioned instances, iterations printed), Theorem contract on the GPU's x."""
    kind, mk = WELL_CONDITIONED[name]
    G = mk()
    s, d = G.numpy()
    eps = EPS[kind]
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=MAX_ITER, step_rule="newton")
    S = solver_for(kind, G, step_rule="newton")
    assert S.solve(eps, MAX_ITER) == "feasible"
    st = S.stats()
    print(f"{name} newton: objective {st['objective']:.10g} (oracle {r.objective:.10g}) iterations "
          f"{st['iters_total']} (oracle {r.iters_total}) evals/iter {st['search_evals'] / max(1, st['iters_total']):.2f}")
    assert abs(st["objective"] - r.objective) <= 1e-6 * abs(r.objective)
    x = S.x().cpu().numpy()
    lp = O.graph_lp(kind, s, d, G.n_vertices, st["bound"])
    assert (lp.C @ x).min() >= 1 - 1e-9
    if not math.isnan(st["certificate"]):
        assert (lp.P @ x).max() == pytest.approx(st["certificate"], rel=1e-9)
