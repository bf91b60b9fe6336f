"""Per-iteration trace of the step search on a BASELINE workload (default c4): accepted alpha and
search passes per MWU iteration of the bench's probe sequence (first outer-bisection bound)."""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--iters", type=int, default=60)
    a = ap.parse_args()
    import torch
    import graphgen as gg
    from bench import WORKLOADS, bracket, graph_stats
    from paper_2307_03307_b200 import Solver
    kind, eps, _ = WORKLOADS[a.workload]
    G = gg.config_graph(a.workload, seed=1, device="cuda")
    gs = graph_stats(G)
    L, H, _ = bracket(kind, gs, eps)
    S = Solver.graph(kind, G.src, G.dst, G.n_vertices, G.n_left if kind == "bmatch" else 0)
    S.probe_begin(math.sqrt(L * H), eps)
    prev = S.scalars()
    for t in range(a.iters):
        out = S.run_iters(1)
        sc = S.scalars()
        print(f"t={int(sc['t'])} alpha={sc['alpha_last']:.6g} k*={math.floor(math.log2(sc['alpha_last'])) + 1 if sc['alpha_last'] >= 1 else 0} "
              f"passes={int(sc['passes'] - prev['passes'])} evals={int(sc['evals'] - prev['evals'])} {out}", flush=True)
        prev = sc
        if out != "running":
            break
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
