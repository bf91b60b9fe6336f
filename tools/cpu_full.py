"""The oracle at FULL BASELINE size on the host cores (one core, pinned): build the explicit LP of a
config from the same seeded generator (CUDA-generated graph copied to the host when a GPU is present,
as bench.py does) and time K oracle MWU iterations at the first outer-bisection bound — the
full-size per-iteration CPU cost the bench's cpu_baseline extrapolates from a reduced instance.
   python tools/cpu_full.py --workload c4 --iters 2     (prints one JSON line)"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--alpha", type=float, default=0.0, help="> 0: fixed step; else Alg. 3")
    a = ap.parse_args()
    import torch
    import graphgen as gg
    import oracle as O
    from bench import WORKLOADS, PinnedCore, bracket, cpu_model, graph_stats
    kind, eps, desc = WORKLOADS[a.workload]
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t0 = time.perf_counter()
    G = gg.config_graph(a.workload, seed=1, device=dev)
    gs = graph_stats(G)
    s, d = G.numpy()
    t_gen = time.perf_counter() - t0
    with PinnedCore(0):
        L, H, _ = bracket(kind, gs, eps)
        B = math.sqrt(L * H)
        t0 = time.perf_counter()
        lp = O.graph_lp(kind, s, d, G.n_vertices, B)
        p = O.Probe(lp, eps)
        t_build = time.perf_counter() - t0
        times = []
        for _ in range(a.iters):
            t0 = time.perf_counter()
            st = p.step(a.alpha if a.alpha > 0 else None)
            times.append(time.perf_counter() - t0)
            if st != O.RUNNING:
                break
    per = sum(times) / len(times)
    print(json.dumps({"workload": f"{a.workload}: {desc}", "kind": kind, "nnz": int(lp.P.nnz + lp.C.nnz),
                      "iterations": len(times), "s_per_iteration": per, "iterations_per_s": 1.0 / per,
                      "step": "fixed alpha" if a.alpha > 0 else "Alg. 3", "build_s": t_build, "generate_s": t_gen,
                      "cores": 1, "pinned_core": 0, "cpu_model": cpu_model(), "host_cores": os.cpu_count()}))


if __name__ == "__main__":
    main()
