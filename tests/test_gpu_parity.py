"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded
inputs — integer structure bit-exact, per-iteration vectors within 1e-10 relative over the
first 50 iterations (fixed and searched steps), full solves within the BASELINE tolerances
(objective 1e-6 relative, same certificate, iterations +-2%)."""
import math

import numpy as np
import pytest
import scipy.sparse as sp
import torch

import graphgen as gg
import oracle as O
from paper_2307_03307_b200.mwu import MwuError
from gpu_common import (assert_vec, csr_tuple, lockstep, lp_mats, self_drift, solver_for)
from instances import FIXED_ORDER_COUNT, MAX_ITER, WELL_CONDITIONED

pytestmark = pytest.mark.gpu

EPS = {"bmatch": 0.1, "match": 0.1, "vcover": 0.05, "domset": 0.05, "densest": 0.1}


def graphs():
    return {
        "bmatch": [gg.bipartite_uniform(200, 300, 5000, seed=3), gg.config_graph("c1"),
                   gg.bipartite_zipf(1024, 1024, 16384, seed=2)],
        "match": [gg.rmat(10, 8, seed=4), gg.hub_graph(6000, 2, 4000, 20000, seed=1)],
        "vcover": [gg.erdos_renyi(2000, 16000, seed=5), gg.hub_graph(6000, 2, 4000, 20000, seed=2)],
        "domset": [gg.rmat(11, 16, seed=6), gg.hub_graph(6000, 2, 4000, 20000, seed=3)],
        "densest": [gg.rmat(10, 16, seed=7), gg.hub_graph(5000, 1, 3000, 15000, seed=4)],
    }


CASES = [(k, i) for k, gl in graphs().items() for i in range(len(gl))]


def _graph(kind, i):
    return graphs()[kind][i]


def _oracle_probe_bound(kind, G):
    """A bound near the optimum: the last feasible probe of the oracle's outer search."""
    s, d = G.numpy()
    r = O.solve(kind, s, d, G.n_vertices, eps=EPS[kind], max_iter=400)
    feas = [p[0] for p in r.probes if p[1] == O.FEASIBLE]
    return (feas[-1] if feas else r.bound), r


# ------------------------------------------------------------------ structure (bit-exact)
@pytest.mark.parametrize("kind,i", CASES)
def test_structure_bit_exact(cuda_ok, kind, i):
    G = _graph(kind, i)
    s, d = G.numpy()
    S = solver_for(kind, G)
    M = O.incidence_M(s, d, G.n_vertices)
    deg = np.diff(M.indptr)
    assert np.array_equal(S.structure("degree").numpy(), deg.astype(np.int32))
    if kind == "domset":
        C = O.closed_neighborhood(s, d, G.n_vertices)
        assert np.array_equal(S.structure("c_rowptr").numpy(), C.indptr.astype(np.int64))
        assert np.array_equal(S.structure("c_colidx").numpy(), C.indices.astype(np.int32))
        return
    if kind in ("bmatch", "match", "densest"):
        # the default (scattered, blocked-order) path builds no vertex -> slot list; the
        # fixed-order engine does
        with pytest.raises(MwuError):
            S.structure("inc_slots")
        S = solver_for(kind, G, deterministic=1)
    rp = S.structure("inc_rowptr").numpy()
    slots = S.structure("inc_slots").numpy().astype(np.uint32)
    assert np.array_equal(rp, M.indptr.astype(np.int64))
    assert np.array_equal((slots >> 1).astype(np.int64), M.indices.astype(np.int64))
    # slot parity b: 0 if the row vertex is src[e], 1 if dst[e]
    rows = np.repeat(np.arange(G.n_vertices), deg)
    e = slots >> 1
    assert np.array_equal(np.where(slots & 1, d[e], s[e]), rows)
    if kind in ("bmatch", "match", "densest"):
        prow = S.structure("prow").numpy()
        _, keep = O.drop_empty_rows(M)
        exp = -np.ones(G.n_vertices, dtype=np.int32)
        exp[keep] = np.arange(keep.size)
        assert np.array_equal(prow, exp)


def test_structure_csr_bit_exact(cuda_ok):
    from paper_2307_03307_b200 import Solver, MIXED
    lp = gg.random_planted_lp(300, 200, 150, 0.03, seed=11)
    P, C = lp_mats(lp)
    # make two empty packing rows (dropped, Q17)
    P = P.tolil(); P[5, :] = 0; P[77, :] = 0; P = P.tocsr(); P.eliminate_zeros()
    S = Solver.csr(MIXED, lp.n, P=csr_tuple(P), C=csr_tuple(C))
    P2, _ = O.drop_empty_rows(P)
    assert np.array_equal(S.structure("p_rowptr").numpy(), P2.indptr)
    assert np.array_equal(S.structure("p_colidx").numpy(), P2.indices)
    Pc, Cc = P2.tocsc(), C.tocsc()
    Pc.sort_indices(); Cc.sort_indices()
    assert np.array_equal(S.structure("pt_rowptr").numpy(), Pc.indptr)
    assert np.array_equal(S.structure("pt_rowidx").numpy(), Pc.indices)
    assert np.array_equal(S.structure("ct_rowptr").numpy(), Cc.indptr)
    assert np.array_equal(S.structure("ct_rowidx").numpy(), Cc.indices)
    assert S.stats()["empty_rows_dropped"] == 2


# ------------------------------------------------------------------ fixed-step parity (T3)
@pytest.mark.parametrize("kind,i", CASES)
def test_fixed_step_parity_alpha_one(cuda_ok, kind, i):
    G = _graph(kind, i)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound(kind, G)
    probe = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), EPS[kind], max_iter=5000)
    S = solver_for(kind, G)
    # standard step: well conditioned, every vector within 1e-10 for 50 iterations
    lockstep(S, probe, B, EPS[kind], 50, alphas=[1.0] * 50, strict_derived=True)


@pytest.mark.parametrize("kind,i", CASES)
def test_fixed_step_parity_oracle_alphas(cuda_ok, kind, i):
    """BASELINE north_star (ii): the oracle's recorded search alphas replayed as fixed steps."""
    G = _graph(kind, i)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound(kind, G)
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    rec = O.Probe(lp, EPS[kind], max_iter=50)
    rec.run()
    alphas = rec.alphas + [1.0] * (50 - len(rec.alphas))
    probe = O.Probe(lp, EPS[kind], max_iter=5000)
    S = solver_for(kind, G)
    n = min(50, max(1, len(rec.alphas)))
    lockstep(S, probe, B, EPS[kind], n, alphas=alphas, drift=self_drift(lp, EPS[kind], alphas, n))


@pytest.mark.parametrize("kind,i", CASES)
def test_search_parity(cuda_ok, kind, i):
    """Alg. 3 on both sides: identical accepted alphas and vectors for 50 iterations."""
    G = _graph(kind, i)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound(kind, G)
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    probe = O.Probe(lp, EPS[kind], max_iter=5000)
    S = solver_for(kind, G)
    lockstep(S, probe, B, EPS[kind], 50, alphas=None, drift=self_drift(lp, EPS[kind], None, 50))


@pytest.mark.parametrize("use_graph", [0, 1])
def test_search_parity_csr_mixed(cuda_ok, use_graph):
    from paper_2307_03307_b200 import Solver, MIXED
    lp = gg.random_planted_lp(400, 250, 180, 0.02, seed=12)
    P, C = lp_mats(lp)
    olp = O.mixed_lp(P, C)
    probe = O.Probe(olp, 0.1, max_iter=5000)
    S = Solver.csr(MIXED, lp.n, P=csr_tuple(P), C=csr_tuple(C), use_graph=use_graph)
    lockstep(S, probe, 1.0, 0.1, 50, alphas=None, drift=self_drift(olp, 0.1, None, 50))


@pytest.mark.parametrize("mode", ["packing", "covering"])
def test_search_parity_csr_pure(cuda_ok, mode):
    from paper_2307_03307_b200 import Solver, PURE_PACKING, PURE_COVERING
    lp = gg.random_planted_lp(300, 220, 160, 0.03, seed=13)
    P, C = lp_mats(lp)
    if mode == "packing":
        ol = O.packing_lp(P, 40.0)
        S = Solver.csr(PURE_PACKING, lp.n, P=csr_tuple(P))
    else:
        ol = O.covering_lp(C, 60.0)
        S = Solver.csr(PURE_COVERING, lp.n, C=csr_tuple(C))
    probe = O.Probe(ol, 0.1, max_iter=5000)
    lockstep(S, probe, 40.0 if mode == "packing" else 60.0, 0.1, 50, alphas=None,
             drift=self_drift(ol, 0.1, None, 50))


# ------------------------------------------------------------------ full solves (T4)
def _contract(S, kind, s, d, nv, st):
    """The returned x satisfies the Theorem's contract on the exact LP."""
    x = S.x().cpu().numpy()
    lp = O.graph_lp(kind, s, d, nv, st["bound"])
    assert (lp.C @ x).min() >= 1 - 1e-9
    if not math.isnan(st["certificate"]):
        assert (lp.P @ x).max() == pytest.approx(st["certificate"], rel=1e-9)
        assert st["max_Px"] == st["certificate"] and st["min_Cx"] == 1.0


@pytest.mark.parametrize("name", sorted(WELL_CONDITIONED))
def test_full_solve_parity(cuda_ok, name):
    """BASELINE full runs, as written: objective within 1e-6 relative of the oracle's, the same
    certificate verdict and probe verdicts, iteration count within +-2%, max_iter = 5000
     — on the instances where the oracle itself is reproducible to that level
    (tests/instances.py; precondition asserted on CPU by test_oracle_conditioning.py).

    densest-bu310 (FIXED_ORDER_COUNT): the default engine sums d^(y) with fp64 atomics, whose
    order changes from run to run; on this instance that alone moves the iteration count by
    -4.4% .. +0.9% between runs of ONE binary (tools/rerun_bu310.py, profiles/rerun_bu310_r2f.log;
    the oracle's own count moves 1.5% under injected rounding noise), so a +-2% assertion on it
    passes or fails by chance.  The +-2% bound is therefore asserted on the fixed-order engine
    (deterministic = 1: 2230 iterations in every run, oracle 2212), and the default engine is held
    to every other full-run tolerance, with its count printed and bounded at 10% as a sanity check
    only."""
    kind, mk = WELL_CONDITIONED[name]
    G = mk()
    s, d = G.numpy()
    eps = EPS[kind]
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=MAX_ITER)

    def run(count_tol, **opts):
        S = solver_for(kind, G, **opts)
        out = S.solve(eps, MAX_ITER)
        st = S.stats()
        print(f"{name} {opts}: objective {st['objective']:.12g} (oracle {r.objective:.12g}) iterations "
              f"{st['iters_total']} (oracle {r.iters_total}) probes {st['probes']} near ties {st['near_tie_count']}")
        assert out == "feasible"
        assert abs(st["objective"] - r.objective) <= 1e-6 * abs(r.objective), (st["objective"], r.objective)
        assert abs(st["bound"] - r.bound) <= 1e-6 * abs(r.bound), (st["bound"], r.bound)
        assert abs(st["iters_total"] - r.iters_total) <= count_tol * r.iters_total, (st["iters_total"], r.iters_total)
        assert st["probes"] == len(r.probes)
        assert (st["certificate"] <= 1 + eps) == (r.certificate <= 1 + eps)
        _contract(S, kind, s, d, G.n_vertices, st)

    if name in FIXED_ORDER_COUNT:
        run(0.02, deterministic=1)
        run(0.10)
    else:
        run(0.02)


@pytest.mark.parametrize("kind,i", CASES)
def test_full_solve_chaotic_diagnostic(cuda_ok, kind, i):
    """Random instances whose searched trajectories are chaotic in fp64 (the oracle's own one-ulp
    reruns disagree by up to 1e-4 in the covering objective and by 10-30% in iterations,
    DESIGN.md §4): the spread is PRINTED, not asserted as parity.  Asserted: the Theorem contract
    on the GPU's x, and that both are (1+eps)-approximations of the same optimum (objectives within
    2 eps of each other)."""
    G = _graph(kind, i)
    s, d = G.numpy()
    eps = EPS[kind]
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=MAX_ITER)
    S = solver_for(kind, G)
    assert S.solve(eps, MAX_ITER) == "feasible"
    st = S.stats()
    print(f"{kind}-{i}: objective {st['objective']:.10g} vs oracle {r.objective:.10g} "
          f"(rel {abs(st['objective'] - r.objective) / abs(r.objective):.2e}); iterations {st['iters_total']} vs "
          f"{r.iters_total}; near ties {st['near_tie_count']}")
    assert abs(st["objective"] - r.objective) <= 2 * eps * abs(r.objective)
    _contract(S, kind, s, d, G.n_vertices, st)


def test_full_solve_csr_mixed(cuda_ok):
    from paper_2307_03307_b200 import Solver, MIXED
    lp = gg.random_planted_lp(500, 300, 200, 0.02, seed=21)
    P, C = lp_mats(lp)
    r = O.solve("mixed", P=P, C=C, eps=0.1)
    S = Solver.csr(MIXED, lp.n, P=csr_tuple(P), C=csr_tuple(C))
    out = S.solve(0.1)
    assert out == r.outcome == "feasible"
    st = S.stats()
    assert st["iters_total"] == r.iters_total
    assert st["certificate"] == pytest.approx(r.certificate, rel=1e-9)
    x = S.x().cpu().numpy()
    assert np.max(np.abs(x - r.x)) <= 1e-9 * np.max(np.abs(r.x))


# ------------------------------------------------------------------ modes and edge cases
def test_graph_and_host_modes_bit_identical(cuda_ok):
    """deterministic=1: every reduction in a fixed order, so the CUDA-graph probe and the
    host-driven loop agree bit for bit."""
    G = gg.rmat(10, 16, seed=9)
    a = solver_for("densest", G, use_graph=1, deterministic=1)
    b = solver_for("densest", G, use_graph=0, deterministic=1)
    a.solve(0.1, 300)
    b.solve(0.1, 300)
    assert a.stats()["iters_total"] == b.stats()["iters_total"]
    assert torch.equal(a.x(), b.x())


@pytest.mark.parametrize("kind", ["vcover", "domset", "bmatch"])
def test_deterministic_path_parity(cuda_ok, kind):
    """The fixed-order (deterministic=1) engine of the other graph kinds under the same lockstep
    checks as the default scattered path."""
    G = _graph(kind, 0)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound(kind, G)
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    probe = O.Probe(lp, EPS[kind], max_iter=5000)
    S = solver_for(kind, G, deterministic=1)
    lockstep(S, probe, B, EPS[kind], 50, alphas=None, drift=self_drift(lp, EPS[kind], None, 50))


@pytest.mark.parametrize("i", [0, 1])
def test_densest_deterministic_path_parity(cuda_ok, i):
    """The fixed-order densest path (deterministic=1: stored v and d^(z), gathered forward
    product) under the same lockstep checks as the default atomic-scatter path."""
    G = _graph("densest", i)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound("densest", G)
    lp = O.graph_lp("densest", s, d, G.n_vertices, B)
    probe = O.Probe(lp, EPS["densest"], max_iter=5000)
    S = solver_for("densest", G, deterministic=1)
    lockstep(S, probe, B, EPS["densest"], 50, alphas=None,
             drift=self_drift(lp, EPS["densest"], None, 50))


def test_densest_fast_path_repeatable_objective(cuda_ok):
    """The atomic-scatter path varies run to run only in summation order: two solves agree on
    the outcome, bound and iteration count of a well-separated instance."""
    G = gg.rmat(10, 16, seed=9)
    a = solver_for("densest", G)
    b = solver_for("densest", G)
    a.solve(0.1, 300)
    b.solve(0.1, 300)
    sa, sb = a.stats(), b.stats()
    assert sa["bound"] == pytest.approx(sb["bound"], rel=1e-6)
    assert sa["probes"] == sb["probes"]


def test_bisect_depth_does_not_change_results(cuda_ok):
    """How many bisection levels a search pass evaluates changes only the pass count, never
    Alg. 3's result (deterministic=1: fixed-order sums, so the comparison is bit-exact)."""
    G = gg.erdos_renyi(3000, 20000, seed=10)
    xs, its = [], []
    for depth in (1, 2, 3):
        S = solver_for("vcover", G, bisect_depth=depth, deterministic=1)
        S.solve(0.05, 500)
        xs.append(S.x())
        its.append(S.stats()["iters_total"])
    assert its[0] == its[1] == its[2]
    assert torch.equal(xs[0], xs[1]) and torch.equal(xs[0], xs[2])


def test_infeasible_csr_and_empty_cover_row(cuda_ok):
    from paper_2307_03307_b200 import Solver, MIXED
    lp = gg.infeasible_lp(6, 0)
    P, C = lp_mats(lp)
    S = Solver.csr(MIXED, lp.n, P=csr_tuple(P), C=csr_tuple(C))
    assert S.solve(0.1) == "infeasible"
    P = sp.csr_matrix(np.eye(2))
    C = sp.csr_matrix(np.array([[1.0, 1.0], [0.0, 0.0]]))
    S = Solver.csr(MIXED, 2, P=csr_tuple(P), C=csr_tuple(C))
    assert S.solve(0.1) == "infeasible"
    assert S.stats()["reason"] == "EMPTY_COVER_ROW"


def test_tight_scalar_instance_matches_oracle(cuda_ok):
    from paper_2307_03307_b200 import Solver, MIXED
    one = sp.csr_matrix(np.array([[1.0]]))
    two = sp.csr_matrix(np.array([[2.0]]))
    S = Solver.csr(MIXED, 1, P=csr_tuple(one), C=csr_tuple(one))
    assert S.solve(0.1) == "infeasible" and S.stats()["reason"] == "MAXD_ZERO"
    S = Solver.csr(MIXED, 1, P=csr_tuple(one), C=csr_tuple(two))
    assert S.solve(0.1) == "feasible"
    assert S.x().item() == 0.5


def test_create_errors(cuda_ok):
    from paper_2307_03307_b200 import Solver, MwuError, MIXED
    with pytest.raises(MwuError, match="self-loop"):
        Solver.graph("vcover", torch.tensor([0, 1]), torch.tensor([0, 2]), 3)
    with pytest.raises(MwuError, match="duplicate"):
        Solver.graph("vcover", torch.tensor([0, 1, 0]), torch.tensor([1, 2, 1]), 3)
    with pytest.raises(MwuError, match="out of range"):
        Solver.graph("match", torch.tensor([0]), torch.tensor([5]), 3)
    with pytest.raises(MwuError, match="BMATCH"):
        Solver.graph("bmatch", torch.tensor([0]), torch.tensor([1]), 4, n_left=2)
    P = sp.csr_matrix(np.array([[1.0, 0.0]]))
    with pytest.raises(MwuError, match="all-zero column"):
        Solver.csr(MIXED, 2, P=csr_tuple(P), C=csr_tuple(P))
    bad = (torch.tensor([0, 2]), torch.tensor([1, 0], dtype=torch.int32), torch.tensor([1.0, 1.0]))
    with pytest.raises(MwuError, match="strictly increasing"):
        Solver.csr(MIXED, 2, P=bad, C=bad)
    neg = (torch.tensor([0, 1]), torch.tensor([0], dtype=torch.int32), torch.tensor([-1.0]))
    with pytest.raises(MwuError, match="negative"):
        Solver.csr(MIXED, 1, P=neg, C=neg)


def test_iter_limit_and_edgeless_domset(cuda_ok):
    G = gg.erdos_renyi(500, 3000, seed=3)
    S = solver_for("vcover", G)
    S.probe_begin(100.0, 0.05)
    p = O.Probe(O.graph_lp("vcover", *G.numpy(), G.n_vertices, 100.0), 0.05)
    assert S.step(1.0) == p.step(1.0)
    S2 = solver_for("vcover", G, max_iter=1)
    S2.probe_begin(150.0, 0.05)
    assert S2.run_probe() in ("iter_limit", "feasible", "infeasible")
    assert S2.scalars()["t"] <= 1
    # edgeless graph: C = I, the dominating-set LP optimum is n (every vertex in the set)
    E = gg.Graph(torch.zeros(0, dtype=torch.int32), torch.zeros(0, dtype=torch.int32), 7)
    S3 = solver_for("domset", E)
    S3.solve(0.05)
    r = O.solve("domset", np.zeros(0, int), np.zeros(0, int), 7, eps=0.05)
    assert S3.stats()["objective"] == pytest.approx(r.objective, rel=1e-6)


def test_host_buffers_e2e(cuda_ok):
    """Inputs from host memory through the same ABI (the e2e path of bench.py)."""
    G = gg.config_graph("c1")
    from paper_2307_03307_b200 import Solver
    S = Solver.graph("bmatch", G.src, G.dst, G.n_vertices, G.n_left)   # CPU tensors
    S.solve(0.1)
    xh = S.x(device="cpu")
    r = O.solve("bmatch", *G.numpy(), G.n_vertices, eps=0.1)
    assert S.stats()["objective"] == pytest.approx(r.objective, rel=1e-6)
    assert xh.device.type == "cpu"


@pytest.mark.parametrize("kind,i,bl,br", [("densest", 0, 6, 5), ("densest", 1, 7, 4), ("bmatch", 2, 5, 6),
                                          ("match", 0, 6, 6), ("match", 1, 8, 5)])
def test_small_block_order_parity(cuda_ok, kind, i, bl, br):
    """The L2-blocked internal edge order with forced small row blocks, so that
    edges cross many (source, destination) block pairs and a warp's 32 edges straddle block
    boundaries (the source-side warp runs restart inside a warp): the same lockstep checks."""
    G = _graph(kind, i)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound(kind, G)
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    probe = O.Probe(lp, EPS[kind], max_iter=5000)
    S = solver_for(kind, G, block_l=bl, block_r=br)
    lockstep(S, probe, B, EPS[kind], 50, alphas=[1.0] * 50, strict_derived=True)


@pytest.mark.parametrize("kind", ["vcover", "match", "densest"])
def test_shuffled_edge_order_parity(cuda_ok, kind):
    """Edge lists in random order (no generator sorting): the warp-segmented source-side sums
    must treat a key that reappears after a different key as a new run (keys A, B, A in one
    warp), in vcover's scatter over the caller's order and in the blocked kinds."""
    G0 = {"vcover": gg.erdos_renyi(2000, 16000, seed=5), "match": gg.rmat(10, 8, seed=4),
          "densest": gg.rmat(10, 16, seed=7)}[kind]
    g = torch.Generator().manual_seed(123)
    perm = torch.randperm(G0.n_edges, generator=g)
    flip = torch.rand(G0.n_edges, generator=g) < 0.5
    src, dst = G0.src[perm], G0.dst[perm]
    src, dst = torch.where(flip, dst, src), torch.where(flip, src, dst)
    G = gg.Graph(src.contiguous(), dst.contiguous(), G0.n_vertices)
    s, d = G.numpy()
    B, _ = _oracle_probe_bound(kind, G)
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    probe = O.Probe(lp, EPS[kind], max_iter=5000)
    S = solver_for(kind, G)
    lockstep(S, probe, B, EPS[kind], 50, alphas=[1.0] * 50, strict_derived=True)


@pytest.mark.parametrize("kind", ["vcover", "domset"])
@pytest.mark.parametrize("compc", [0, 1])
def test_compact_covering_rows_parity(cuda_ok, kind, compc):
    """The search over compacted covering records plus the inactive aggregate (default for
    vcover / domset on one rank) and over the dense rows (compact_cover = 0): both
    under the lockstep checks against the oracle, on both graphs of the kind."""
    for i in (0, 1):
        G = _graph(kind, i)
        s, d = G.numpy()
        B, _ = _oracle_probe_bound(kind, G)
        lp = O.graph_lp(kind, s, d, G.n_vertices, B)
        probe = O.Probe(lp, EPS[kind], max_iter=5000)
        S = solver_for(kind, G, compact_cover=compc)
        lockstep(S, probe, B, EPS[kind], 50, alphas=None, drift=self_drift(lp, EPS[kind], None, 50))


def test_inputs_produced_on_a_side_stream(cuda_ok):
    """mwu_options.stream: the edge list is produced asynchronously on a torch side stream behind a
    long sleep kernel; create (called with that stream current) must wait for it — the structure
    equals the one built from the finished list — and the output copy lands on that stream too."""
    from paper_2307_03307_b200 import Solver
    G = gg.rmat(12, 16, seed=9)
    ref = solver_for("vcover", G).structure("degree")
    side = torch.cuda.Stream()
    src_h, dst_h = G.src.pin_memory(), G.dst.pin_memory()
    with torch.cuda.stream(side):
        torch.cuda._sleep(200_000_000)                       # ~0.1 s of GPU time before the copies
        src = src_h.to("cuda", non_blocking=True)
        dst = dst_h.to("cuda", non_blocking=True)
        S = Solver.graph("vcover", src, dst, G.n_vertices)  # options.stream = side
        deg = S.structure("degree")
        S.solve(0.05, 200)
        x = S.x()
    side.synchronize()
    assert torch.equal(deg, ref)
    assert x.abs().sum().item() > 0
