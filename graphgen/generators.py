"""Seeded graph / LP generators (torch; CPU for small cases, CUDA for full size).

Recipes follow SURVEY.md §8(d) "Concrete synthetic inputs" and BASELINE.json
configs (BJ:7-11).  The paper's own inputs (SuiteSparse graphs, Graph500 kron,
rgg; Table 1) are not available; these synthetic graphs
stand in for them (R-MAT with a,b,c,d = .57,.19,.19,.05 is the Graph500 recipe
behind the paper's kron-X graphs).

Every generator is deterministic for a given (seed, device type).  A CUDA- and
a CPU-generated instance with the same seed differ; tests always take both
sides' inputs from one generated instance.

Edge-list conventions: edge id e = position in the returned list;
general graphs store each undirected edge once with src < dst, lists sorted by
(src, dst); bipartite graphs put left vertices at [0, n_left) and right
vertices at [n_left, n_vertices), sorted by (left, right).
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass
class Graph:
    src: torch.Tensor          # int32 [E]
    dst: torch.Tensor          # int32 [E]
    n_vertices: int
    n_left: int = 0            # > 0: bipartite, left ids [0, n_left)
    name: str = ""

    @property
    def n_edges(self) -> int:
        return int(self.src.numel())

    def to(self, device) -> "Graph":
        return Graph(self.src.to(device), self.dst.to(device), self.n_vertices,
                     self.n_left, self.name)

    def numpy(self):
        return self.src.cpu().numpy(), self.dst.cpu().numpy()


@dataclasses.dataclass
class CsrLP:
    """A general positive LP  P x <= 1, C x >= 1, x >= 0  in CSR form (int64 rowptr)."""
    n: int
    p_rowptr: torch.Tensor | None
    p_col: torch.Tensor | None
    p_val: torch.Tensor | None
    c_rowptr: torch.Tensor | None
    c_col: torch.Tensor | None
    c_val: torch.Tensor | None
    name: str = ""


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _finish(a: torch.Tensor, b: torch.Tensor, n: int, n_left: int, name: str) -> Graph:
    return Graph(a.to(torch.int32).contiguous(), b.to(torch.int32).contiguous(), int(n), int(n_left), name)


# --------------------------------------------------------------------------- c1
def bipartite_uniform(n_left: int, n_right: int, n_edges: int, seed: int = 1, device="cpu") -> Graph:
    """BJ:7 c1: n_edges distinct (left, right) pairs sampled uniformly without replacement.

    key k drawn without replacement from [0, n_left*n_right); l = k // n_right,
    r = n_left + k % n_right; sorted by (l, r).
    """
    g = _gen(seed, device)
    total = n_left * n_right
    if n_edges > total:
        raise ValueError("more edges than pairs")
    if total <= (1 << 26):
        keys = torch.randperm(total, generator=g, device=device)[:n_edges]
    else:  # rejection: oversample, dedup, random subset
        keys = torch.empty(0, dtype=torch.int64, device=device)
        while keys.numel() < n_edges:
            k = int((n_edges - keys.numel()) * 1.2) + 1024
            keys = torch.unique(torch.cat([keys, torch.randint(0, total, (k,), generator=g, device=device)]))
        keys = keys[torch.randperm(keys.numel(), generator=g, device=device)[:n_edges]]
    keys, _ = torch.sort(keys)
    return _finish(keys // n_right, n_left + keys % n_right, n_left + n_right, n_left,
                   f"bipartite_uniform({n_left}+{n_right},{n_edges})")


# --------------------------------------------------------------------------- c2
def erdos_renyi(n: int, m: int, seed: int = 1, device="cpu") -> Graph:
    """BJ:8 c2: G(n, m) — m distinct unordered pairs u<v, no self-loops (rejection + dedup)."""
    g = _gen(seed, device)
    keys = torch.empty(0, dtype=torch.int64, device=device)
    while keys.numel() < m:
        k = int((m - keys.numel()) * 1.05) + 1024
        u = torch.randint(0, n, (k,), generator=g, device=device, dtype=torch.int64)
        v = torch.randint(0, n, (k,), generator=g, device=device, dtype=torch.int64)
        keep = u != v
        a, b = torch.minimum(u, v)[keep], torch.maximum(u, v)[keep]
        keys = torch.unique(torch.cat([keys, a * n + b]))
    if keys.numel() > m:
        keys = keys[torch.randperm(keys.numel(), generator=g, device=device)[:m]]
        keys, _ = torch.sort(keys)
    return _finish(keys // n, keys % n, n, 0, f"erdos_renyi({n},{m})")


# ------------------------------------------------------------------------ c3/c4
def rmat(scale: int, edge_factor: int = 16, a=0.57, b=0.19, c=0.19, seed: int = 1, device="cpu",
         chunk: int = 1 << 26) -> Graph:
    """BJ:9/BJ:10 c3/c4: R-MAT (Graph500 recipe, no noise, no relabel), symmetrized,
    self-loops dropped, duplicates removed.  edge_factor * 2^scale samples; per level
    r < a -> (0,0), < a+b -> (0,1), < a+b+c -> (1,0), else (1,1)."""
    g = _gen(seed, device)
    n = 1 << scale
    n_samples = edge_factor * n
    keys = []
    for start in range(0, n_samples, chunk):
        k = min(chunk, n_samples - start)
        u = torch.zeros(k, dtype=torch.int64, device=device)
        v = torch.zeros(k, dtype=torch.int64, device=device)
        for _ in range(scale):
            r = torch.rand(k, generator=g, device=device, dtype=torch.float64)
            bu = (r >= a + b).to(torch.int64)                              # quadrants (1,0),(1,1)
            bv = ((r >= a) & (r < a + b)).to(torch.int64) | (r >= a + b + c).to(torch.int64)
            u = u * 2 + bu
            v = v * 2 + bv
            del r, bu, bv
        keep = u != v
        lo, hi = torch.minimum(u, v)[keep], torch.maximum(u, v)[keep]
        keys.append(torch.unique(lo * n + hi))
        del u, v, keep, lo, hi
    keys = torch.unique(torch.cat(keys))
    return _finish(keys // n, keys % n, n, 0, f"rmat(s={scale},ef={edge_factor})")


# --------------------------------------------------------------------------- c5
def zipf_truncated_cap(s: float = 1.5, mean: float = 16.0) -> int:
    """Smallest cap K with E[deg] >= mean for deg ~ Zipf(s) truncated to [1, K]."""
    num = den = 0.0
    k = 0
    while True:
        k += 1
        w = k ** (-s)
        num += k * w
        den += w
        if num / den >= mean:
            return k


def bipartite_zipf(n_left: int, n_right: int, n_edges: int, s: float = 1.5, seed: int = 1,
                   device="cpu") -> Graph:
    """BJ:11 c5 (reading SURVEY Q20): right-vertex degrees i.i.d. Zipf(s) truncated to [1, K]
    with K the smallest cap giving mean >= n_edges/n_right, adjusted by +-1 on random right
    vertices to total exactly n_edges; each right vertex gets distinct uniform left endpoints;
    edges sorted by (left, right)."""
    g = _gen(seed, device)
    K = zipf_truncated_cap(s, n_edges / n_right)
    ks = torch.arange(1, K + 1, dtype=torch.float64, device=device)
    cdf = torch.cumsum(ks ** (-s), 0)
    cdf = cdf / cdf[-1]
    deg = torch.searchsorted(cdf, torch.rand(n_right, generator=g, device=device, dtype=torch.float64)) + 1
    deg = deg.clamp_(1, K).to(torch.int64)
    diff = n_edges - int(deg.sum())
    while diff != 0:
        elig = torch.nonzero(deg < min(K, n_left) if diff > 0 else deg > 1).flatten()
        pick = elig[torch.randperm(elig.numel(), generator=g, device=device)[:abs(diff)]]
        deg[pick] += 1 if diff > 0 else -1
        diff = n_edges - int(deg.sum())
    rights = torch.repeat_interleave(torch.arange(n_right, dtype=torch.int64, device=device), deg)
    lefts = torch.randint(0, n_left, (n_edges,), generator=g, device=device, dtype=torch.int64)
    while True:  # resample left endpoints that repeat within one right vertex
        key = rights * n_left + lefts
        skey, order = torch.sort(key)
        dup_sorted = torch.zeros_like(skey, dtype=torch.bool)
        dup_sorted[1:] = skey[1:] == skey[:-1]
        ndup = int(dup_sorted.sum())
        del skey, key
        if ndup == 0:
            del order, dup_sorted
            break
        idx = order[dup_sorted]
        lefts[idx] = torch.randint(0, n_left, (ndup,), generator=g, device=device, dtype=torch.int64)
        del order, dup_sorted, idx
    key = lefts * n_right + rights
    del lefts, rights
    key, _ = torch.sort(key)
    return _finish(key // n_right, n_left + key % n_right, n_left + n_right, n_left,
                   f"bipartite_zipf({n_left}+{n_right},{n_edges},s={s})")


# ------------------------------------------------------------- small families
def _from_pairs(pairs, n, n_left=0, name="") -> Graph:
    if len(pairs) == 0:
        z = torch.zeros(0, dtype=torch.int32)
        return Graph(z, z.clone(), n, n_left, name)
    t = torch.tensor(sorted(tuple(p) for p in pairs), dtype=torch.int64)
    return _finish(t[:, 0], t[:, 1], n, n_left, name)


def complete_graph(n: int) -> Graph:
    return _from_pairs([(i, j) for i in range(n) for j in range(i + 1, n)], n, 0, f"K{n}")


def complete_bipartite(a: int, b: int) -> Graph:
    return _from_pairs([(i, a + j) for i in range(a) for j in range(b)], a + b, a, f"K{a},{b}")


def star_graph(leaves: int) -> Graph:
    return _from_pairs([(0, j) for j in range(1, leaves + 1)], leaves + 1, 0, f"S{leaves}")


def path_graph(n: int) -> Graph:
    return _from_pairs([(i, i + 1) for i in range(n - 1)], n, 0, f"P{n}")


def cycle_graph(n: int) -> Graph:
    return _from_pairs([(min(i, (i + 1) % n), max(i, (i + 1) % n)) for i in range(n)], n, 0, f"C{n}")


def circulant_regular(n: int, k: int) -> Graph:
    """k-regular circulant graph on n vertices (k even: offsets 1..k/2; k odd needs n even: + n/2)."""
    offs = list(range(1, k // 2 + 1))
    pairs = set()
    for i in range(n):
        for o in offs:
            j = (i + o) % n
            pairs.add((min(i, j), max(i, j)))
        if k % 2:
            j = (i + n // 2) % n
            pairs.add((min(i, j), max(i, j)))
    return _from_pairs(sorted(pairs), n, 0, f"circ({n},{k})")


def random_small_graph(n: int, p: float, seed: int) -> Graph:
    g = _gen(seed, "cpu")
    r = torch.rand(n, n, generator=g, dtype=torch.float64)
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if r[i, j] < p]
    return _from_pairs(pairs, n, 0, f"gnp({n},{p},{seed})")


def random_small_bipartite(a: int, b: int, p: float, seed: int) -> Graph:
    g = _gen(seed, "cpu")
    r = torch.rand(a, b, generator=g, dtype=torch.float64)
    pairs = [(i, a + j) for i in range(a) for j in range(b) if r[i, j] < p]
    return _from_pairs(pairs, a + b, a, f"bip({a},{b},{p},{seed})")


def hub_graph(n: int, hubs: int, hub_deg: int, extra: int, seed: int = 1) -> Graph:
    """Graph with `hubs` vertices of degree >= hub_deg (long rows, > one seg tile) plus `extra`
    random edges; exercises the long-row path of the segmented kernels."""
    g = _gen(seed, "cpu")
    keys = []
    for h in range(hubs):
        nb = torch.randperm(n, generator=g)[:hub_deg + 1]
        nb = nb[nb != h][:hub_deg]
        a, b = torch.minimum(nb, torch.tensor(h)), torch.maximum(nb, torch.tensor(h))
        keys.append(a * n + b)
    u = torch.randint(0, n, (extra,), generator=g)
    v = torch.randint(0, n, (extra,), generator=g)
    keep = u != v
    keys.append(torch.minimum(u, v)[keep] * n + torch.maximum(u, v)[keep])
    k = torch.unique(torch.cat(keys))
    return _finish(k // n, k % n, n, 0, f"hub({n},{hubs},{hub_deg},{extra})")


def rgg(scale: int, avg_degree: float = 10.0, seed: int = 1) -> Graph:
    """Random geometric graph: 2^scale points uniform in the unit square (numpy PCG64
    `default_rng(seed)`), an edge between every pair closer than r with pi r^2 n = avg_degree —
    the family of the paper's rgg-X inputs (e.g. rgg-18 of Table 3), which are not
    in the container.  Edges (u < v) sorted."""
    import numpy as np
    n = 1 << scale
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = math.sqrt(avg_degree / (math.pi * n))
    nc = max(1, int(1.0 / r))
    cell = np.minimum((pts * nc).astype(np.int64), nc - 1)
    cid = cell[:, 0] * nc + cell[:, 1]
    order = np.argsort(cid, kind="stable")
    cs = cid[order]
    start = np.searchsorted(cs, np.arange(nc * nc), "left")
    end = np.searchsorted(cs, np.arange(nc * nc), "right")
    us, vs = [], []
    for dx, dy in ((0, 0), (0, 1), (1, -1), (1, 0), (1, 1)):
        tx, ty = cell[:, 0] + dx, cell[:, 1] + dy
        ok = (tx >= 0) & (tx < nc) & (ty >= 0) & (ty < nc)
        src = np.nonzero(ok)[0]
        t = tx[src] * nc + ty[src]
        cnt = end[t] - start[t]
        rep_src = np.repeat(src, cnt)
        offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
        dst = order[np.repeat(start[t], cnt) + offs]
        keep = (np.sum((pts[rep_src] - pts[dst]) ** 2, axis=1) < r * r) & (rep_src != dst)
        if dx == 0 and dy == 0:
            keep &= rep_src < dst
        us.append(rep_src[keep])
        vs.append(dst[keep])
    u, v = np.concatenate(us), np.concatenate(vs)
    a, b = np.minimum(u, v), np.maximum(u, v)
    k = np.unique(a * n + b)
    return _finish(torch.from_numpy(k // n), torch.from_numpy(k % n), n, 0, f"rgg-{scale}")


def biadjacency(g: Graph) -> Graph:
    """Bipartite graph read from the adjacency matrix of g (rows = left copy, columns = right copy):
    the paper's bmatch reading of a general matrix; both directions of every edge."""
    n = g.n_vertices
    a = torch.cat([g.src, g.dst]).to(torch.int64)
    b = torch.cat([g.dst, g.src]).to(torch.int64) + n
    k, _ = torch.sort(a * (2 * n) + b)
    return _finish(k // (2 * n), k % (2 * n), 2 * n, n, f"biadj({g.name})")


def gmatch_instance(n_users: int, n_items: int, seed: int = 1, deg_lo: int = 10, deg_hi: int = 40,
                    s: float = 1.0, user_bounds=(3.0, 5.0), item_ub: float = 200.0):
    """Synthetic generalized-matching instance shaped like the paper's App. A.2 preprocessing of
    the Netflix / KDD ratings graphs (the datasets are not in the container): a
    bipartite users x items graph, every user with deg_lo..deg_hi ratings (users with < 10 are
    excluded there) of items drawn with Zipf(s) popularity, bounds lb = 3, ub = 5 per user and
    no lower, upper item_ub per item.  Returns (Graph, lb, ub) with float64 bound tensors."""
    import numpy as np
    rng = np.random.default_rng(seed)
    w = 1.0 / np.arange(1, n_items + 1) ** s
    w /= w.sum()
    src, dst = [], []
    for u in range(n_users):
        k = int(rng.integers(deg_lo, deg_hi + 1))
        items = rng.choice(n_items, size=min(k, n_items), replace=False, p=w)
        src.extend([u] * len(items))
        dst.extend((n_users + items).tolist())
    o = np.lexsort((np.asarray(dst), np.asarray(src)))
    g = Graph(torch.tensor(np.asarray(src)[o], dtype=torch.int32), torch.tensor(np.asarray(dst)[o], dtype=torch.int32),
              n_users + n_items, n_users, f"gm({n_users},{n_items},{seed})")
    lb = torch.zeros(n_users + n_items, dtype=torch.float64)
    ub = torch.full((n_users + n_items,), float(item_ub), dtype=torch.float64)
    lb[:n_users] = user_bounds[0]
    ub[:n_users] = user_bounds[1]
    return g, lb, ub


def disjoint_union(*graphs: Graph) -> Graph:
    """Vertex-disjoint union, edges in the order of the parts (ids shifted per part)."""
    src, dst, off = [], [], 0
    for g in graphs:
        src.append(g.src.to(torch.int64) + off)
        dst.append(g.dst.to(torch.int64) + off)
        off += g.n_vertices
    return _finish(torch.cat(src), torch.cat(dst), off, 0, "U(" + ";".join(g.name for g in graphs) + ")")


def plus_random_edges(g: Graph, k: int, seed: int) -> Graph:
    """g plus k extra distinct random edges (numpy PCG64 `default_rng(seed)`, appended in draw
    order, endpoints as drawn) — a perturbed copy of a structured graph."""
    import numpy as np
    rng = np.random.default_rng(seed)
    s, d = g.numpy()
    have = set(zip(s.tolist(), d.tolist())) | set(zip(d.tolist(), s.tolist()))
    S, D = list(s), list(d)
    while k:
        a, b = rng.integers(0, g.n_vertices, 2)
        if a != b and (a, b) not in have:
            have.add((a, b))
            have.add((b, a))
            S.append(a)
            D.append(b)
            k -= 1
    return Graph(torch.tensor(S, dtype=torch.int32), torch.tensor(D, dtype=torch.int32), g.n_vertices, 0,
                 f"{g.name}+{len(S) - len(s)}r{seed}")


# ---------------------------------------------------------- general CSR LPs
def _random_csr(rows: int, n: int, density: float, g, lo=0.5, hi=2.0, min_per_row=1):
    mask = torch.rand(rows, n, generator=g, dtype=torch.float64) < density
    for r in range(rows):  # guarantee non-empty rows
        if int(mask[r].sum()) < min_per_row:
            mask[r, torch.randint(0, n, (min_per_row,), generator=g)] = True
    vals = lo + (hi - lo) * torch.rand(rows, n, generator=g, dtype=torch.float64)
    return torch.where(mask, vals, torch.zeros_like(vals))


def _dense_to_csr(A: torch.Tensor):
    rows, cols = torch.nonzero(A, as_tuple=True)
    counts = torch.bincount(rows, minlength=A.shape[0])
    rowptr = torch.zeros(A.shape[0] + 1, dtype=torch.int64)
    rowptr[1:] = torch.cumsum(counts, 0)
    return rowptr, cols.to(torch.int32), A[rows, cols].contiguous()


def random_planted_lp(n: int, m_p: int, m_c: int, density: float, seed: int) -> CsrLP:
    """Feasible-by-design positive LP (SPEC S:330 property suite): plant x* > 0, then
    scale each packing row so (P x*)_j in [0.5, 1] and each covering row so (C x*)_j in [1, 2].
    Every column of P gets a nonzero (P:272 init needs ||P_{:,i}||_inf > 0)."""
    g = _gen(seed, "cpu")
    xs = 0.5 + torch.rand(n, generator=g, dtype=torch.float64)
    P = _random_csr(m_p, n, density, g)
    for i in range(n):
        if not bool((P[:, i] > 0).any()):
            P[torch.randint(0, m_p, (1,), generator=g), i] = 1.0
    C = _random_csr(m_c, n, density, g)
    tp = 0.5 + 0.5 * torch.rand(m_p, generator=g, dtype=torch.float64)
    tc = 1.0 + torch.rand(m_c, generator=g, dtype=torch.float64)
    P = P * (tp / (P @ xs))[:, None]
    C = C * (tc / (C @ xs))[:, None]
    pr, pc, pv = _dense_to_csr(P)
    cr, cc, cv = _dense_to_csr(C)
    return CsrLP(n, pr, pc, pv, cr, cc, cv, f"planted({n},{m_p},{m_c},{seed})")


def infeasible_lp(n: int, seed: int) -> CsrLP:
    """Infeasible by construction: packing rows x_i <= 1/2 (P = 2I) and one covering row
    (1/n) sum x >= 1 (needs mean x >= 1)."""
    P = 2.0 * torch.eye(n, dtype=torch.float64)
    C = torch.full((1, n), 1.0 / n, dtype=torch.float64)
    pr, pc, pv = _dense_to_csr(P)
    cr, cc, cv = _dense_to_csr(C)
    return CsrLP(n, pr, pc, pv, cr, cc, cv, f"infeasible({n})")


# ------------------------------------------------------------- BJ configs
CONFIGS = {
    # name: (kind, eps, description)                             BASELINE.json line
    "c1": ("bmatch", 0.1, "bipartite uniform 1000+1000, 10,000 edges"),      # BJ:7
    "c2": ("vcover", 0.05, "Erdos-Renyi n=2^20, avg degree 16"),              # BJ:8
    "c3": ("domset", 0.05, "R-MAT scale 22, edge factor 16"),                 # BJ:9
    "c4": ("densest", 0.1, "R-MAT scale 24, edge factor 16"),                 # BJ:10
    "c5": ("bmatch", 0.1, "bipartite Zipf(1.5) 2^26+2^26, 2^30 edges"),      # BJ:11
}


def config_graph(name: str, scale_down: int = 0, seed: int = 1, device="cpu") -> Graph:
    """The graph of config `name`; scale_down > 0 gives the same-recipe reduced instance
    (vertex counts divided by 2^scale_down, average degree kept)."""
    sd = int(scale_down)
    if name == "c1":
        return bipartite_uniform(1000, 1000, 10_000, seed=seed, device=device)
    if name == "c2":
        n = 1 << (20 - sd)
        return erdos_renyi(n, 8 * n, seed=seed, device=device)
    if name == "c3":
        return rmat(22 - sd, 16, seed=seed, device=device)
    if name == "c4":
        return rmat(24 - sd, 16, seed=seed, device=device)
    if name == "c5":
        side = 1 << (26 - sd)
        return bipartite_zipf(side, side, 16 * side, seed=seed, device=device)
    raise KeyError(name)


def _selfcheck():  # pragma: no cover - manual use
    print(zipf_truncated_cap(1.5, 16.0), math.log(2))
