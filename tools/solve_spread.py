"""Oracle full-solve conditioning survey (how tests/instances.py WELL_CONDITIONED
was chosen): for candidate instances of a graph kind, run the oracle's full solve (max_iter 5000)
from x0 and from x0 scaled by 1 +- 2^-52 and print the objective / iteration spreads and whether
any probe ended at the iteration cap.  CPU only.   python tools/solve_spread.py <kind>"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import graphgen as gg  # noqa: E402
import oracle as O  # noqa: E402

EPS = {"bmatch": 0.1, "match": 0.1, "vcover": 0.05, "domset": 0.05, "densest": 0.1}
K = gg.complete_bipartite
U = gg.disjoint_union


def candidates(kind):
    c = []
    if kind == "bmatch":
        c += [(f"bu300x400s{s}", lambda s=s: gg.bipartite_uniform(300, 400, 3000, seed=s)) for s in range(20, 30)]
        c += [(f"bz256s{s}", lambda s=s: gg.bipartite_zipf(256, 256, 2048, seed=s)) for s in range(3)]
        c += [("c1", lambda: gg.config_graph("c1"))]
    elif kind == "match":
        c += [(f"er2000s{s}", lambda s=s: gg.erdos_renyi(2000, 8000, seed=s)) for s in range(20, 28)]
        c += [(f"rmat9s{s}", lambda s=s: gg.rmat(9, 4, seed=30 + s)) for s in range(3)]
    elif kind == "densest":
        c += [(f"er300s{s}", lambda s=s: gg.erdos_renyi(300, 1500, seed=70 + s)) for s in range(8)]
        c += [(f"rmat8s{s}", lambda s=s: gg.rmat(8, 8, seed=80 + s)) for s in range(6)]
        c += [(f"K{a},{b}", lambda a=a, b=b: K(a, b)) for a, b in ((10, 20), (15, 40), (7, 50))]
    else:   # vcover, domset
        c += [(f"K{a},{b}", lambda a=a, b=b: K(a, b)) for a, b in ((10, 20), (15, 40), (25, 26), (5, 200))]
        c += [(f"er200s{s}", lambda s=s: gg.erdos_renyi(200, 2000, seed=110 + s)) for s in range(3)]
        c += [("S50+K8,12", lambda: U(gg.star_graph(50), K(8, 12))),
              ("K20,30+5", lambda: gg.plus_random_edges(K(20, 30), 5, 1)),
              ("U(K6;K8;C9)", lambda: U(gg.complete_graph(6), gg.complete_graph(8), gg.cycle_graph(9))),
              ("path101", lambda: gg.path_graph(101))]
    return c


def main(kind):
    for name, mk in candidates(kind):
        G = mk()
        s, d = G.numpy()
        t0 = time.time()
        rs = [O.solve(kind, s, d, G.n_vertices, eps=EPS[kind], max_iter=5000, x0_scale=sc)
              for sc in (1.0, 1 + 2.0 ** -52, 1 - 2.0 ** -52)]
        r = rs[0]
        print(json.dumps(dict(
            kind=kind, name=name, n=G.n_vertices, E=G.n_edges, objective=r.objective,
            obj_spread=max(abs(q.objective - r.objective) / abs(r.objective) for q in rs[1:]),
            iters=r.iters_total, iters_spread=max(abs(q.iters_total - r.iters_total) for q in rs[1:]),
            capped=sum(1 for q in rs for p in q.probes if p[1] == O.ITER_LIMIT),
            probes="".join(p[1][0] for p in r.probes), probe_iters=[p[2] for p in r.probes],
            secs=round(time.time() - t0, 1))), flush=True)


if __name__ == "__main__":
    main(sys.argv[1])
