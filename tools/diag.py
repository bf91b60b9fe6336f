#!/usr/bin/env python
"""Diagnostics on a BJ workload (GPU): per-iteration alpha, search passes, and the fraction of
active rows (d^(y) > 0, d^(z) > 0, d > 0).  Also the driver for ncu captures (use_graph=0 so the
kernels are ordinary launches)."""
import argparse, math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import graphgen as gg
from paper_2307_03307_b200 import Solver
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--scale-down", type=int, default=0)
ap.add_argument("--iters", type=int, default=12)
ap.add_argument("--use-graph", type=int, default=0)
ap.add_argument("--active", type=int, default=1)
ap.add_argument("--phases", type=int, default=0)
ap.add_argument("--bound", type=float, default=0.0, help="probe bound (default: the first outer bisection bound)")
ap.add_argument("--block-r", type=int, default=0)
ap.add_argument("--skip", type=int, default=0, help="iterations run through the probe graph before the listed ones")
a = ap.parse_args()
kind, eps, _ = bench.WORKLOADS[a.workload]
G = gg.config_graph(a.workload, scale_down=a.scale_down, seed=1, device="cuda")
gs = bench.graph_stats(G)
S = Solver.graph(kind, G.src, G.dst, G.n_vertices, G.n_left if kind == "bmatch" else 0, use_graph=a.use_graph,
                 block_r=a.block_r)
L, H, _ = bench.bracket(kind, gs, eps)
B = a.bound if a.bound > 0 else math.sqrt(L * H)
S.probe_begin(B, eps)
if a.skip > 0:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    S.run_iters(a.skip)        # use_graph=0 context: host-driven, but no per-iteration printing
    torch.cuda.synchronize()
    print(f"skipped {a.skip} iterations in {time.perf_counter() - t0:.1f} s", flush=True)
print("stats", {k: v for k, v in S.stats().items() if k in ("n", "m_P", "m_C", "nnz_P", "nnz_C")}, "B", B, flush=True)
for t in range(a.iters):
    sc0 = S.scalars()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    if a.phases:
        pr = S.profile_iters(1)
        out = "running" if S.scalars()["t"] > sc0["t"] and pr["iters"] > 0 else "stopped"
    else:
        out = S.run_iters(1)
    torch.cuda.synchronize(); el = time.perf_counter() - t0
    sc = S.scalars()
    line = f"t={int(sc['t'])} out={out} alpha={sc['alpha_last']:.6g} passes={sc['passes']-sc0['passes']:.0f} evals={sc['evals']-sc0['evals']:.0f} ms={1000*el:.2f}"
    if a.phases:
        line += " | " + " ".join(f"{k}={pr[k]['ms']:.3f}" for k in ("column", "step", "search", "update"))
    if a.active:
        fr = {}
        for k in ("d", "dy", "dz"):
            try:
                v = S.vec(k)
                fr[k] = float((v > 0).double().mean())
            except Exception:
                pass
        line += " active " + " ".join(f"{k}={v:.3f}" for k, v in fr.items())
    print(line, flush=True)
    if out != "running":
        break
