"""Multi-GPU layer: edge-sharded iteration with one allreduce of the
scattered forward product per iteration plus allgathered phase reductions.

CPU (`-m "not gpu"`): the shard ranges tile the edge list, the unique-id distribution over a
world-size-2 gloo group (the same code path graph_distributed uses with NCCL), and the two exchange
patterns (edge-sharded forward product, row-sharded transposed product: partial scatter + one
allreduce) over that group against the oracle's incidence product.
GPU: the sharded engine with an in-process rank group on one device (SimGroup: one host thread
per rank, host barriers, no kernel waits on another) against the single-GPU engine and the
oracle: fixed-step vectors within 1e-10 relative, identical searched solves."""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import graphgen as gg
import oracle as O


# ---------------------------------------------------------------------------------- CPU
@pytest.mark.parametrize("E,W", [(0, 1), (1, 4), (10, 3), (1000003, 8), (2 ** 30, 8), (260380362, 7)])
def test_shard_ranges_tile_the_edges(E, W):
    from paper_2307_03307_b200 import mwu
    prev = 0
    sizes = []
    for r in range(W):
        a, b = mwu.shard_range(E, W, r)
        assert a == prev and b >= a
        sizes.append(b - a)
        prev = b
    assert prev == E
    assert max(sizes) - min(sizes) <= 2 * 1024          # ranges on MWU_CT = 1024-edge tile boundaries


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, E, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_03307_b200 import mwu
    uid = mwu.share_unique_id(lambda: bytes(range(128)))      # stands in for ncclGetUniqueId
    a, b = mwu.shard_range(E, world, rank)
    t = torch.tensor([a, b], dtype=torch.int64)
    g = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(g, t)
    out[rank] = (uid, [tuple(x.tolist()) for x in g])
    dist.destroy_process_group()


def test_unique_id_and_ranges_over_gloo():
    world, E = 2, 123457
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gloo_worker, args=(world, port, E, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == bytes(range(128))
    ranges = res[0][1]
    assert ranges == res[1][1]
    assert ranges[0][0] == 0 and ranges[-1][1] == E and ranges[0][1] == ranges[1][0]


def _gloo_exchange_worker(rank, world, port, out):
    """The sharded engine's two exchange patterns over a real process group: the
    edge-sharded matching forward product d^(y) = M d (each rank scatters its mwu_shard_range of
    the edges, one allreduce of the row vector), and the row-sharded vertex-cover transposed
    product h = M w (each rank's covering rows, one allreduce of the length-n gradient)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2307_03307_b200 import mwu
    G = gg.bipartite_zipf(700, 900, 5003, seed=4)              # same seeded graph on every rank
    src, dst = G.src.numpy().astype(np.int64), G.dst.numpy().astype(np.int64)
    E, n = len(src), G.n_vertices
    rng = np.random.default_rng(11)
    d = rng.random(E)                                          # one value per edge (variable / covering row)
    e0, e1 = mwu.shard_range(E, world, rank)
    part = np.zeros(n)
    np.add.at(part, src[e0:e1], d[e0:e1])
    np.add.at(part, dst[e0:e1], d[e0:e1])
    t = torch.from_numpy(part)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    cnt = torch.tensor([e1 - e0], dtype=torch.int64)
    dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
    out[rank] = (t.numpy().copy(), int(cnt.item()), (e0, e1))
    dist.destroy_process_group()


def test_sharded_products_over_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_gloo_exchange_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    G = gg.bipartite_zipf(700, 900, 5003, seed=4)
    src, dst = G.src.numpy(), G.dst.numpy()
    M = O.incidence_M(src, dst, G.n_vertices)                  # vertices x edges
    d = np.random.default_rng(11).random(len(src))
    want = O.matvec(M, d)
    assert res[0][1] == res[1][1] == len(src)                   # the ranges cover every edge once
    assert res[0][2][1] == res[1][2][0]
    for r in range(world):
        np.testing.assert_allclose(res[r][0], want, rtol=1e-13, atol=0)
    np.testing.assert_array_equal(res[0][0], res[1][0])         # every rank holds the same reduced vector


# ---------------------------------------------------------------------------------- GPU
def _run_ranks(world, fn):
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # pragma: no cover - reported below
            errs.append((r, e))
    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if any(t.is_alive() for t in th):
        raise RuntimeError("a rank did not finish")
    if errs:
        raise errs[0][1]
    return out


def _solver(kind, G, **kw):
    from paper_2307_03307_b200 import Solver
    return Solver.graph(kind, G.src.cuda(), G.dst.cuda(), G.n_vertices, G.n_left if kind == "bmatch" else 0, **kw)


CASES = [("densest", gg.rmat(10, 16, seed=7), 0.1), ("bmatch", gg.bipartite_zipf(1024, 1024, 16384, seed=2), 0.1),
         ("match", gg.hub_graph(6000, 2, 4000, 20000, seed=1), 0.1),
         ("vcover", gg.erdos_renyi(5000, 40000, seed=5), 0.05), ("domset", gg.rmat(12, 16, seed=6), 0.05)]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("ci", range(len(CASES)))
def test_sharded_fixed_steps_match_oracle(cuda_ok, world, ci):
    """Sharded engine (W ranks as in-process contexts on one device), 20 standard steps
    (alpha = 1): every rank holds the same whole vectors, within 1e-10 relative of
    the ORACLE's independent run and of the single-GPU engine."""
    from paper_2307_03307_b200.mwu import SimGroup
    kind, G, eps = CASES[ci]
    s, d = G.numpy()
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=300)
    B = [p[0] for p in r.probes if p[1] == O.FEASIBLE][-1]
    probe = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), eps)
    for _ in range(20):
        assert probe.step(1.0) == O.RUNNING
    ora = {"x": probe.x, "y": probe.y, "z": probe.z, "d": probe.last["d"], "dy": probe.last["dy"],
           "dz": probe.last["dz"], "wc": probe.v / probe.SC}
    one = _solver(kind, G)
    one.probe_begin(B, eps)
    for _ in range(20):
        one.step(1.0)
    keys = ("x", "y", "z", "d", "dy", "dz", "wc")
    ref = {k: one.vec(k).cpu().numpy() for k in keys}
    grp = SimGroup(world)

    def rank_fn(rk):
        S = _solver(kind, G, world=world, rank=rk, comm_group=grp)
        S.probe_begin(B, eps)
        for _ in range(20):
            S.step(1.0)
        return {k: S.vec(k).cpu().numpy() for k in keys}
    outs = _run_ranks(world, rank_fn)
    grp.close()

    def rel(a, b):
        return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))
    sig = probe.sigma
    for o in outs:
        for k in ("x", "y", "z", "wc"):
            assert rel(o[k], ora[k]) <= 1e-10, (k, "oracle", rel(o[k], ora[k]))
            assert rel(o[k], ref[k]) <= 1e-10, (k, "1 GPU", rel(o[k], ref[k]))
        # d, d^(y), d^(z): 1e-10 plus the 1 - g/h cancellation allowance (a few ulps of g/h times
        # sigma x, as in the single-GPU strict lockstep)
        allow = 1e-12 * sig * np.abs(probe.x)
        for k, al in (("d", allow), ("dy", probe.lp.P @ allow), ("dz", probe.lp.C @ allow)):
            assert np.all(np.abs(o[k] - ora[k]) <= 1e-10 * np.abs(ora[k]) + al), (k, "oracle")
    for o in outs[1:]:
        for k in ref:
            assert np.array_equal(o[k], outs[0][k])          # every rank holds the same vectors


# densest is left out: no densest instance keeps its iteration count within 2% under rounding noise
# with margin (bu310: 1.5% for the oracle's own reruns, 2.4% measured sharded); the sharded densest
# engine is held to 1e-10 against the oracle by the fixed-step test above
SHARDED_WELL = ["bmatch-bu21", "match-er21", "vcover-K5,200", "domset-K25,26", "domset-K20,30+5"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", SHARDED_WELL)
def test_sharded_solve(cuda_ok, name):
    """Full sharded solve (W = 2) on the well-conditioned instances (tests/instances.py): the
    BASELINE full-run tolerances against the ORACLE and the single-GPU engine — objective and
    bound within 1e-6 relative, iterations within +-2%, identical probe count."""
    from paper_2307_03307_b200.mwu import SimGroup
    from instances import EPS, MAX_ITER, WELL_CONDITIONED
    kind, mk = WELL_CONDITIONED[name]
    G = mk()
    eps = EPS[kind]
    s, d = G.numpy()
    r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=MAX_ITER)
    one = _solver(kind, G)
    one.solve(eps, MAX_ITER)
    st1 = one.stats()
    grp = SimGroup(2)

    def rank_fn(rk):
        S = _solver(kind, G, world=2, rank=rk, comm_group=grp)
        out = S.solve(eps, MAX_ITER)
        return out, S.stats(), S.x().cpu().numpy()
    outs = _run_ranks(2, rank_fn)
    grp.close()
    (o0, st0, x0), (o1, stb, x1) = outs
    assert o0 == o1 == "feasible"
    assert np.array_equal(x0, x1)
    assert st0["bound"] == stb["bound"] and st0["probes"] == stb["probes"]
    for ref_obj, ref_bound, ref_its, ref_probes in ((r.objective, r.bound, r.iters_total, len(r.probes)),
                                                    (st1["objective"], st1["bound"], st1["iters_total"], st1["probes"])):
        assert abs(st0["objective"] - ref_obj) <= 1e-6 * abs(ref_obj), (st0["objective"], ref_obj)
        assert abs(st0["bound"] - ref_bound) <= 1e-6 * abs(ref_bound), (st0["bound"], ref_bound)
        assert abs(st0["iters_total"] - ref_its) <= 0.02 * ref_its, (st0["iters_total"], ref_its)
        assert st0["probes"] == ref_probes
    lp = O.graph_lp(kind, s, d, G.n_vertices, st0["bound"])
    assert (lp.C @ x0).min() >= 1 - 1e-9                      # Theorem contract on the exact LP


@pytest.mark.gpu
@pytest.mark.parametrize("ci", range(len(CASES)))
def test_nccl_plumbing_one_rank(cuda_ok, ci):
    """The NCCL communicator (dlopen'ed library, unique id through torch.distributed, allreduce
    and allgather on the library's stream) driving the sharded engine with one rank: the same
    iterates as the plain engine over 15 standard steps, and 12 searched iterations with the
    collectives captured into the probe's CUDA graph (conditional WHILE nodes, device-side
    Alg. 3 control, no host round trip per search pass) against the host-driven sharded loop
    (in-process group of one rank): identical step sizes, iterates within 1e-10.  (The fast
    paths reduce with fp64 atomics, so two runs agree to rounding, not bit for bit.  Several
    ranks need several GPUs; the sharding itself is covered by the SimGroup tests above.)"""
    from paper_2307_03307_b200 import Solver
    from paper_2307_03307_b200.mwu import SimGroup
    port = _free_port()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        kind, G, eps = CASES[ci]
        s, d = G.numpy()
        r = O.solve(kind, s, d, G.n_vertices, eps=eps, max_iter=300)
        B = [p[0] for p in r.probes if p[1] == O.FEASIBLE][-1]
        one = _solver(kind, G)
        nl = G.n_left if kind == "bmatch" else 0
        S = Solver.graph_distributed(kind, G.src.cuda(), G.dst.cuda(), G.n_vertices, nl)
        for T in (one, S):
            T.probe_begin(B, eps)
            for _ in range(15):
                T.step(1.0)
        for k in ("x", "y", "z", "d", "dy"):
            a, b = S.vec(k).cpu().numpy(), one.vec(k).cpu().numpy()
            assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= 1e-10, k
        grp = SimGroup(1)
        H = _solver(kind, G, world=1, rank=0, comm_group=grp)
        alphas = []
        for T in (S, H):
            T.probe_begin(B, eps)
            T.run_iters(12)
            alphas.append(T.scalars()["alpha_last"])
        assert S.stats()["probe_graph"] == 1                # NCCL collectives inside the graph
        assert H.stats()["probe_graph"] == 0                # host-driven reference
        assert S.scalars()["t"] == H.scalars()["t"] and alphas[0] == alphas[1]
        for k in ("x", "y", "z"):
            a, b = S.vec(k).cpu().numpy(), H.vec(k).cpu().numpy()
            assert np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)) <= 1e-10, k
        out = S.solve(eps, 300)
        assert out == "feasible" and S.stats()["probe_graph"] == 1
        del H
        grp.close()
    finally:
        dist.destroy_process_group()
