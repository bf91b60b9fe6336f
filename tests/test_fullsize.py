"""Parity at BASELINE.json's full sizes (c2-c5), in the launch configuration bench.py times
(default fast path, CUDA-graph probe, the bench's first outer bound): after three graph-launched
iterations, one more iteration is stepped with g, h recorded and every phase is checked against
the oracle's definitions —

* sampled outputs the oracle computes one by one on the CPU (math.fsum over the incident
  entries of the LP built from the paper's definitions): g, h (1e-10 relative),
  the direction d (bit-exact from the GPU's own g, h, x), the forward products d^(y), d^(z)
  (1e-10), the updates of x, y, z (bit-exact);
* properties that hold at any size: the weights w_p, w_c sum to 1 and are the normalised
  exponentials of the cached y, z (ratios on samples), and Alg. 3 (oracle.binsearch on the full
  cached vectors) returns exactly the GPU's step size.

c1 (10^4 edges) is covered at full size by the element-by-element tests of test_gpu_parity.py.
"""
import math

import numpy as np
import pytest
import torch

import bench
import graphgen as gg
import oracle as O

pytestmark = pytest.mark.gpu
RT = 1e-10
NS = 1500     # sampled variables / rows


def _rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.fixture(autouse=True)
def _free_device_memory():
    yield
    import gc
    gc.collect()
    torch.cuda.empty_cache()


def _setup(workload):
    """The bench's first outer bound (or, if that probe ends within three iterations, the next
    bounds of the bisection towards the feasible end)."""
    from paper_2307_03307_b200 import Solver
    kind, eps, _ = bench.WORKLOADS[workload]
    G = gg.config_graph(workload, seed=1, device="cuda")
    gs = bench.graph_stats(G)
    L, H, sense = bench.bracket(kind, gs, eps)
    S = Solver.graph(kind, G.src, G.dst, G.n_vertices, G.n_left if kind == "bmatch" else 0)
    B = math.sqrt(L * H)
    for _ in range(6):
        S.probe_begin(B, eps)
        if S.run_iters(3) == "running":
            break
        B = math.sqrt(B * (H if sense < 0 else L))
    else:
        pytest.fail("no probe of the bisection stays running for three iterations")
    S.set_record(True)
    return kind, eps, G, S, B


def _snap(S, keys):
    return {k: S.vec(k) for k in keys}


def _incident(G, verts):
    """Edges incident to the sampled vertices (torch selection on the device, sums on the CPU)."""
    v = torch.as_tensor(verts, device=G.src.device, dtype=torch.int32)
    m = torch.isin(G.src, v) | torch.isin(G.dst, v)
    e = torch.nonzero(m).flatten()
    return e.cpu().numpy(), G.src[e].cpu().numpy(), G.dst[e].cpu().numpy()


def _np(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("workload", ["c4", "c5", "c2", "c3"])
def test_full_size_phase_parity(cuda_ok, workload):
    kind, eps, G, S, B = _setup(workload)
    rng = np.random.default_rng(7)
    n = S.n
    vs = np.unique(rng.integers(0, n, NS))

    def smp(t, idx):
        return t[torch.as_tensor(idx, device=t.device)].cpu().numpy()

    # only samples (and the row vectors Alg. 3 needs) leave the device; full edge-length
    # vectors are dropped as soon as they are sampled (c5: 8.6 GB each)
    t = S.vec("x"); x0 = smp(t, vs); del t
    y0, z0, wp, wc = (_np(S.vec(k)) for k in ("y", "z", "wp", "wc"))
    sc = S.scalars()
    S.step(0.0)
    alpha = S.scalars()["alpha_last"]
    t = S.vec("g"); g = smp(t, vs); del t
    t = S.vec("h"); h = smp(t, vs); del t
    dvec = S.vec("d")
    dv = smp(dvec, vs)
    dy, dz = _np(S.vec("dy")), _np(S.vec("dz"))
    t = S.vec("x"); x1 = smp(t, vs); del t
    y1, z1 = _np(S.vec("y")), _np(S.vec("z"))
    sigma, invB = sc["sigma"], 1.0 / B
    pd = {"d": dvec}

    # weights: normalised, and the exponentials of the cached rows (shift-free ratios)
    for w in (wp, wc):
        assert abs(float(np.sum(w)) - 1.0) <= 1e-12
    for vec, w, sgn in ((y0, wp, 1.0), (z0, wc, -1.0)):
        if vec.size > 1:
            j = int(np.argmax(w))
            for a in rng.integers(0, vec.size, NS):
                ref = math.exp(sgn * sc["eta"] * (vec[a] - vec[j]))
                assert abs(w[a] / w[j] - ref) <= 1e-9 * ref + 1e-300
    src = G.src.cpu().numpy()
    dst = G.dst.cpu().numpy()
    prow = S.structure("prow").numpy() if kind in ("bmatch", "densest") else None
    # ---- transposed products g, h and the direction on sampled variables
    if kind == "densest":
        for k, s_ in enumerate(vs):
            e, b = s_ >> 1, s_ & 1
            vtx = src[e] if b == 0 else dst[e]
            assert _rel(g[k], (1.0 / B) * wp[prow[vtx]]) <= RT
            assert _rel(h[k], wc[e]) <= RT
    elif kind == "bmatch":
        for k, e in enumerate(vs):
            assert _rel(g[k], math.fsum([wp[prow[src[e]]], wp[prow[dst[e]]]])) <= RT
            assert h[k] == invB
    else:   # pure covering: g = 1/M, h = C^T w_c
        assert np.all(g == invB)
        es, esrc, edst = _incident(G, vs)
        terms = {int(v): ([] if kind == "vcover" else [wc[v]]) for v in vs}
        for e, a, b in zip(es, esrc, edst):
            if kind == "vcover":          # C = M^T: row e holds x_a + x_b
                for v in (a, b):
                    if int(v) in terms:
                        terms[int(v)].append(wc[e])
            else:                         # C = I + A, symmetric
                if int(a) in terms:
                    terms[int(a)].append(wc[b])
                if int(b) in terms:
                    terms[int(b)].append(wc[a])
        for k, v in enumerate(vs):
            assert _rel(h[k], math.fsum(terms[int(v)])) <= RT
    assert np.array_equal(dv, O.direction(g, h, x0, sigma))
    # ---- forward products on sampled rows
    if kind in ("densest", "bmatch"):
        mP = dy.size
        inv = np.full(mP, -1, dtype=np.int64)
        inv[prow[prow >= 0]] = np.nonzero(prow >= 0)[0]
        rows = rng.integers(0, mP, NS // 3)
        verts = inv[rows]
        es, esrc, edst = _incident(G, verts)
        slots = np.concatenate([2 * es, 2 * es + 1]) if kind == "densest" else es
        dmap = dict(zip(slots.tolist(), smp(pd["d"], slots).tolist())) if slots.size else {}
        terms = {int(v): [] for v in verts}
        for e, a, b in zip(es, esrc, edst):
            for side, v in ((0, a), (1, b)):
                if int(v) in terms:
                    terms[int(v)].append((1.0 / B) * dmap[2 * e + side] if kind == "densest" else dmap[e])
        for r, v in zip(rows, verts):
            assert _rel(dy[r], math.fsum(terms[int(v)])) <= RT
        if kind == "densest":
            es2 = rng.integers(0, dz.size, NS)
            assert np.array_equal(dz[es2], smp(pd["d"], 2 * es2) + smp(pd["d"], 2 * es2 + 1))    # W d
        else:
            assert _rel(dz[0], float(torch.sum(pd["d"]).item()) * invB) <= 1e-12                  # (1/M) 1^T d
    else:
        assert _rel(dy[0], float(torch.sum(pd["d"]).item()) * invB) <= 1e-12
        rows = rng.integers(0, dz.size, NS)
        if kind == "vcover":
            assert np.array_equal(dz[rows], smp(pd["d"], src[rows]) + smp(pd["d"], dst[rows]))
        else:
            es, esrc, edst = _incident(G, rows)
            nb = np.unique(np.concatenate([rows, esrc, edst]))
            dmap = dict(zip(nb.tolist(), smp(pd["d"], nb).tolist()))
            terms = {int(v): [dmap[int(v)]] for v in rows}
            for a, b in zip(esrc, edst):
                if int(a) in terms:
                    terms[int(a)].append(dmap[int(b)])
                if int(b) in terms:
                    terms[int(b)].append(dmap[int(a)])
            for v in rows:
                assert _rel(dz[v], math.fsum(terms[int(v)])) <= RT
    # ---- Alg. 3 on the full cached vectors gives the GPU's alpha exactly
    si = O.SearchInputs(y0, dy, z0, dz, sc["eta"], sc["sP"], sc["SP"], sc["sC"], sc["SC"], wp, wc)
    assert alpha == O.binsearch(si, eps, "prose").alpha
    # ---- updates, same operation order: bit-exact
    assert np.array_equal(x1, x0 + alpha * dv)
    ry = rng.integers(0, y0.size, NS)
    assert np.array_equal(y1[ry], y0[ry] + alpha * dy[ry])
    rz = rng.integers(0, z0.size, NS)
    assert np.array_equal(z1[rz], z0[rz] + alpha * dz[rz])
