#!/usr/bin/env python
"""bench.py — MWU iterations/s (+ nnz/s, HBM-roofline fraction) of the B200 hot path.

A "step" is one MWU iteration (Alg. 2 loop body P:663-682: column, forward products, Alg. 3
search passes, update) of the solve's own probe sequence: probes start at the first outer
bisection bound (Q14) and follow the bisection when a probe terminates, exactly as mwu_solve
does.  Default workload: BASELINE config c4 (densest subgraph, R-MAT scale 24, eps 0.1) — the
largest single-GPU-only configuration.  See DESIGN.md §5 for the byte accounting.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1..c5] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (kind, eps, description)                                   BASELINE.json
    "c1": ("bmatch", 0.1, "bipartite uniform 1000+1000, 10,000 edges"),          # configs[0]
    "c2": ("vcover", 0.05, "Erdos-Renyi n=2^20, avg degree 16"),                  # configs[1]
    "c3": ("domset", 0.05, "R-MAT scale 22, edge factor 16, C = I + A"),          # configs[2]
    "c4": ("densest", 0.1, "R-MAT scale 24, edge factor 16, Charikar dual"),      # configs[3]
    "c5": ("bmatch", 0.1, "bipartite Zipf(1.5) 2^26+2^26, 2^30 edges"),          # configs[4]
}
CPU_SAMPLE_SCALEDOWN = {"c1": 0, "c2": 5, "c3": 8, "c4": 9, "c5": 10}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


def graph_stats(G):
    import torch
    deg = torch.bincount(torch.cat([G.src, G.dst]).long(), minlength=G.n_vertices)
    return dict(E=G.n_edges, nv=G.n_vertices, nprime=int((deg > 0).sum()), maxdeg=int(deg.max()))


def bracket(kind, gs, eps):
    """Q14 bracket end points (the same formulas mwu_solve uses) for the first probe bound."""
    E, nv, npr, D = gs["E"], gs["nv"], gs["nprime"], gs["maxdeg"]
    if kind == "densest":
        return E / npr, D / 2.0, -1
    if kind in ("bmatch", "match"):
        return E / D, float(E), +1
    if kind == "vcover":
        return E / D, float(npr), -1
    if kind == "domset":
        return nv / (D + 1), float(nv), -1
    raise KeyError(kind)


def phase_credits(kind, st):
    """Split of the algorithmic bytes of one MWU iteration (mwu_stats.bytes_alg_per_iter
    B_alg = S_fwd + S_tr + 32 n + 40 (m_P' + m_C')) over the phase kernels of our fused design: each
    term goes to the ONE kernel that moves that data first, so the credits sum to B_alg exactly.
    S = S_fwd + S_tr (structure of the four products; S_fwd = S_tr), rows: 8 B each for d^(.) write,
    y (z) read, d^(.) read, y (z) write and the weight gather.  Embedded singleton rows cost 0.
      densest / matching: the column kernel applies O^T / M^T AND scatters d^(y) = P d (fused),
                          reads/writes x and d (32 n), writes d^(y) and gathers u (16 m_P), and for
                          densest also the covering rows' z read/write, d^(z) write, v (32 m_C);
                          search: y, d^(y) read (16 m_P) + d^(z) read (8 m_C); update: y write (8 m_P)
      vcover / domset:    column = S/2 + 32 n + v gather (8 m_C); step (forward product + record
                          compaction) = S/2 + d^(z) write + z read (16 m_C); search = d^(z) read
                          (8 m_C); update = z write (8 m_C)."""
    balg, n = st["bytes_alg_per_iter"], st["n"]
    mP = st["m_P"] if st["m_P"] > 1 else 0          # embedded singleton rows: 0 bytes
    mC = st["m_C"] if st["m_C"] > 1 else 0
    S = balg - 32.0 * n - 40.0 * (mP + mC)
    if kind in ("densest", "bmatch", "match"):
        c = {"column": S + 32.0 * n + 16.0 * mP + 32.0 * mC, "step": 0.0, "search": 16.0 * mP + 8.0 * mC,
             "update": 8.0 * mP}
    else:
        c = {"column": S / 2 + 32.0 * n + 8.0 * mC, "step": S / 2 + 16.0 * mC, "search": 8.0 * mC + 16.0 * mP,
             "update": 8.0 * mC + 8.0 * mP}
    assert abs(sum(c.values()) - balg) <= 1e-6 * balg, (c, balg)
    return c


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.out = ""

    def summary(self):
        rows = [r.split(",") for r in (self.out or "").strip().splitlines() if r.strip()]
        sm, mx, reasons = [], 0.0, set()
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
            except (ValueError, IndexError):
                continue
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(workload, phase):
    """DRAM bytes per launch of the phase's dominant kernel from the committed ncu --set full
    summary (profiles/ncu_traffic.json, written from the captures under gpurun_out/)."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        e = t[workload][phase]
        return e["dram_bytes_per_launch"], e
    except Exception:
        return None, None


def measured_peak_gbs():
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(mp["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- CPU oracle
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class PinnedCore:
    """Run the oracle pinned to one host core (taskset -c <core> equivalent) and single-threaded
    BLAS, then restore the affinity: the CPU baseline states exactly the cores it used."""

    def __init__(self, core=0):
        self.core = core

    def __enter__(self):
        self.saved = os.sched_getaffinity(0)
        try:
            os.sched_setaffinity(0, {self.core})
        except OSError:
            pass
        return self

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.saved)


def cpu_oracle_rate(workload, seed, seconds=15.0, min_iters=3, steps=None):
    """The oracle as it stands, single process pinned to one core (numpy/scipy, one thread of
    compute), on the same-recipe reduced instance of `workload`; returns iterations/s scaled to
    the full workload by the nonzero ratio (the per-iteration work is linear in nnz)."""
    with PinnedCore(0):
        return _cpu_oracle_rate(workload, seed, seconds, min_iters, steps)


def _cpu_oracle_rate(workload, seed, seconds=15.0, min_iters=3, steps=None):
    import numpy as np  # noqa: F401

    import graphgen as gg
    import oracle as O
    kind, eps, _ = WORKLOADS[workload]
    sd = CPU_SAMPLE_SCALEDOWN[workload]
    G = gg.config_graph(workload, scale_down=sd, seed=seed)
    s, d = G.numpy()
    gs = graph_stats(G)
    L, H, _ = bracket(kind, gs, eps)
    B = math.sqrt(L * H)
    lp = O.graph_lp(kind, s, d, G.n_vertices, B)
    nnz = lp.P.nnz + lp.C.nnz
    sense = -1 if kind in ("densest", "vcover", "domset") else +1
    p = O.Probe(lp, eps, max_iter=10 ** 9)
    t0 = time.perf_counter()
    it = 0
    while True:
        st = p.step()
        if st != O.RUNNING:      # next bisection probe, as the solver would
            ok = st == O.FEASIBLE
            if (ok and sense > 0) or (not ok and sense < 0):
                L = B
            else:
                H = B
            B = math.sqrt(L * H)
            p = O.Probe(O.graph_lp(kind, s, d, G.n_vertices, B), eps, max_iter=10 ** 9)
            continue
        it += 1
        el = time.perf_counter() - t0
        if steps is not None and it >= steps:
            break
        if steps is None and el >= seconds and it >= min_iters:
            break
    el = time.perf_counter() - t0
    return it / el, nnz, it, el, f"{G.name} (config {workload} recipe at 1/2^{sd} scale), {it} MWU iterations in {el:.1f}s"


def full_nnz(kind, gs):
    E, nv = gs["E"], gs["nv"]
    if kind == "densest":
        return 4 * E
    if kind in ("bmatch", "match"):
        return 3 * E
    if kind == "vcover":
        return 2 * E + nv
    if kind == "domset":
        return nv + 2 * E + nv
    raise KeyError(kind)


def run_reference(args):
    ws, rk, _ = dist_env()
    if rk != 0:
        return 0
    import graphgen as gg
    kind, eps, desc = WORKLOADS[args.workload]
    # full-size nnz for scaling the sampled rate (counted from the generator's recipe on CPU
    # would be slow at scale; use the same GPU-free count as the main arm when available)
    gs_full = json.loads(os.environ.get("MWU_BENCH_GS", "null") or "null")
    if gs_full is None:
        gs_full = approx_full_stats(args.workload)
    cpu_it = cpu_oracle_rate(args.workload, args.seed, steps=args.warmup)
    rate, nnz_s, it, el, sample = cpu_oracle_rate(args.workload, args.seed, steps=args.steps)
    value = rate * nnz_s / full_nnz(kind, gs_full)
    line = {
        "impl": "reference", "metric": "MWU iterations/s", "value": value, "unit": "iterations/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.workload}: {desc}", "kind": kind, "eps": eps},
        "cpu_baseline": {"value": value, "unit": "iterations/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "pinned_core": 0, "host_cores": os.cpu_count()},
        "e2e": {"value": value, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    del cpu_it
    print(json.dumps(line))
    return 0


def approx_full_stats(workload):
    """Shape of the full-size instance measured on the generator (seed 1) — SURVEY §8(d)."""
    table = {
        "c1": dict(E=10000, nv=2000, nprime=2000, maxdeg=23),
        "c2": dict(E=8388608, nv=1 << 20, nprime=1 << 20, maxdeg=40),
        "c3": dict(E=64154589, nv=1 << 22, nprime=(1 << 22) - 1798548, maxdeg=162984),
        "c4": dict(E=260380362, nv=1 << 24, nprime=8871146, maxdeg=405783),
        "c5": dict(E=1 << 30, nv=1 << 27, nprime=1 << 27, maxdeg=435),
    }
    return table[workload]


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch

    import graphgen as gg
    from paper_2307_03307_b200 import Solver, build as B
    ws, rk, lr = dist_env()
    torch.cuda.set_device(lr)
    if ws > 1 or args.shard:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    B.build()
    kind, eps, desc = WORKLOADS[args.workload]
    t0 = time.perf_counter()
    G = gg.config_graph(args.workload, seed=args.seed, device="cuda")
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    gs = graph_stats(G)
    # c4 / c5 shard their edges (one allreduce of d^(y) per iteration), c2 / c3 their covering
    # rows (one allreduce of the column gradient per iteration); c1 (10^4 edges)
    # runs one replica per GPU
    sharded = (ws > 1 or args.shard) and args.workload in ("c2", "c3", "c4", "c5")
    make = Solver.graph_distributed if sharded else Solver.graph
    opts = dict(max_iter=args.max_iter, block_l=args.block_l, block_r=args.block_r)
    S = make(kind, G.src, G.dst, G.n_vertices, G.n_left if kind == "bmatch" else 0, **opts)
    st0 = S.stats()
    L, H, sense = bracket(kind, gs, eps)

    state = {"L": L, "H": H, "B": math.sqrt(L * H), "probes": 0}
    S.probe_begin(state["B"], eps)

    def next_probe(outcome):
        ok = outcome == "feasible"
        if (ok and sense > 0) or (not ok and sense < 0):
            state["L"] = state["B"]
        else:
            state["H"] = state["B"]
        if state["H"] <= (1 + eps / 4) * state["L"]:      # solve finished: restart the sequence
            state["L"], state["H"] = L, H
        state["B"] = math.sqrt(state["L"] * state["H"])
        state["probes"] += 1
        S.probe_begin(state["B"], eps)

    window = {"phase_ms": {p: 0.0 for p in ("column", "step", "search", "update")}, "passes": 0.0}

    def run_steps(k, account=False):
        done = 0
        while done < k:
            sc0 = S.scalars()
            ph0 = S.stats()["t_phase_ms"]
            out = S.run_iters(k - done)
            sc1 = S.scalars()
            done += int(sc1["t"] - sc0["t"])
            if account:        # device-side phase times (%globaltimer, inside the graph) of these steps
                ph1 = S.stats()["t_phase_ms"]
                for p in window["phase_ms"]:
                    window["phase_ms"][p] += ph1[p] - ph0[p]
                window["passes"] += sc1["passes"] - sc0["passes"]
            if out != "running":
                next_probe(out)
        return done

    run_steps(args.warmup)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = None
    with Clocks(lr) as clk:
        e0.record()
        n_done = run_steps(args.steps, account=True)
        e1.record()
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del launches0
    # per-phase profile (host-driven, CUDA events around each phase) on the same probe sequence
    prof = None
    for _ in range(8):
        prof = S.profile_iters(args.profile_iters)
        if prof["iters"] > 0:
            break
        next_probe(S.run_iters(1))       # probe already terminated: follow the bisection
    stats = S.stats()
    if rk != 0:
        return 0
    value = (1 if sharded else ws) * n_done / (ms / 1000.0)
    nnz_iter = full_nnz(kind, gs)
    credit = phase_credits(kind, stats)
    peak, peak_kind = measured_peak_gbs()
    phases = {}
    for ph in ("column", "step", "search", "update"):
        p = prof[ph]
        if p["launches"] > 0 and p["ms"] > 0:
            ms_iter = p["ms"] / prof["iters"]                       # all launches of the phase per iteration
            dram, _ = ncu_traffic(args.workload, ph)                # ncu DRAM bytes per launch (committed summary)
            per_launch = p["launches"] / prof["iters"]
            phases[ph] = {"ms_per_iter": ms_iter, "launches_per_iter": per_launch,
                          "alg_bytes_per_iter": credit[ph], "alg_gbs": credit[ph] / (ms_iter / 1000.0) / 1e9,
                          "ncu_dram_bytes_per_iter": None if dram is None else dram * (prof["passes"] / prof["iters"] if ph == "search" else 1.0)}
            if phases[ph]["ncu_dram_bytes_per_iter"] is not None:
                phases[ph]["ncu_dram_gbs"] = phases[ph]["ncu_dram_bytes_per_iter"] / (ms_iter / 1000.0) / 1e9
    dom = max(phases, key=lambda k: phases[k]["ms_per_iter"])
    launches_per_iter = sum(prof[p]["launches"] for p in ("column", "step", "search", "update")) / max(1, prof["iters"])
    passes_per_iter = prof["passes"] / max(1, prof["iters"])
    # whole-iteration roofline against the credited algorithmic bytes (SURVEY §8d B_alg)
    balg = stats["bytes_alg_per_iter"]
    ms_per_step = ms / n_done
    cpu = None
    if not args.no_cpu and ws == 1:
        rate, nnz_s, it, el, sample = cpu_oracle_rate(args.workload, args.seed, seconds=args.cpu_seconds)
        cpu = {"value": rate * nnz_s / nnz_iter, "unit": "iterations/s", "cores": 1, "kind": "oracle",
               "sample": sample + f"; rate scaled to the full workload by nnz ({nnz_s:,} -> {nnz_iter:,})",
               "nnz_per_s": rate * nnz_s, "cpu_model": cpu_model(), "pinned_core": 0,
               "host_cores": os.cpu_count()}
    # e2e: the public API from pinned host buffers: create (H2D of the edge list) + K steps +
    # D2H of x_out, device-timed
    e2e = None
    if not args.no_e2e:
        src_h = G.src.cpu().pin_memory()
        dst_h = G.dst.cpu().pin_memory()
        x_h = torch.empty(S.n, dtype=torch.float64).pin_memory()
        del S
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        S2 = make(kind, src_h, dst_h, G.n_vertices, G.n_left if kind == "bmatch" else 0, **opts)
        S2.probe_begin(math.sqrt(L * H), eps)
        S = S2
        state.update({"L": L, "H": H, "B": math.sqrt(L * H)})
        n2 = run_steps(args.steps)
        from paper_2307_03307_b200.mwu import lib, _ptr, _check
        _check(lib().mwu_get_vec(S2._h, 0, _ptr(x_h), S2.n), S2._h)
        f1.record()
        torch.cuda.synchronize()
        ms2 = f0.elapsed_time(f1)
        e2e = {"value": (1 if sharded else ws) * n2 / (ms2 / 1000.0), "unit": "iterations/s",
               "h2d_bytes_per_step": int(8 * gs["E"] / max(1, n2)), "d2h_bytes_per_step": int(8 * S2.n / max(1, n2)),
               "note": f"create from pinned host edge list + {n2} steps + x to pinned host, {ms2:.1f} ms"}
    line = {
        "metric": "MWU iterations/s", "value": value, "unit": "iterations/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {desc}", "kind": kind, "eps": eps, "seed": args.seed,
                   "n_vars": stats["n"], "m_P": stats["m_P"], "m_C": stats["m_C"], "nnz": nnz_iter,
                   "edges": gs["E"], "first_bound": math.sqrt(L * H),
                   "l2": "inputs larger than L2 (per-vector GBs)",
                   "parallelism": ((f"edge-sharded x{ws} (NCCL allreduce of d^(y) per iteration)"
                                    if kind in ("densest", "bmatch") else
                                    f"row-sharded x{ws} (NCCL allreduce of the column gradient per iteration)")
                                   if sharded else (f"replicas x{ws}" if ws > 1 else "1 GPU"))},
        "nnz_per_s": nnz_iter * value,
        "iteration_roofline": {"bytes_alg_per_iter": balg, "achieved_gbs": balg / (ms_per_step / 1000) / 1e9,
                               "frac_of_8TBs": balg / (ms_per_step / 1000) / 8e12,
                               "frac_of_measured": balg / (ms_per_step / 1000) / 1e9 / peak},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": phases[dom]["alg_gbs"], "peak": peak, "unit": "GB/s",
                     "frac": phases[dom]["alg_gbs"] / peak, "traffic": ncu_traffic(args.workload, dom)[0],
                     "traffic_gbs": phases[dom].get("ncu_dram_gbs"),
                     "traffic_frac": (phases[dom]["ncu_dram_gbs"] / peak) if phases[dom].get("ncu_dram_gbs") else None,
                     "note": "achieved = the kernel's share of B_alg per iteration / its CUDA-event time (it credits x, d "
                             "of every edge; the kernel skips those of edges inactive in this and the last step); "
                             "traffic = ncu dram__bytes_read+write per launch",
                     "traffic_source": (ncu_traffic(args.workload, dom)[1] or {}).get("source"),
                     "peak_source": peak_kind},
        "phases": phases, "search_passes_per_iter": passes_per_iter,
        "timed_window": {"phase_ms_per_iter": {p: v / max(1, n_done) for p, v in window["phase_ms"].items()},
                         "search_passes_per_iter": window["passes"] / max(1, n_done),
                         "note": "device-side phase times of the timed graph-launched iterations (%globaltimer at "
                                 "each phase end, launch gaps included); `phases` is a host-driven profile of the "
                                 "iterations after the window"},
        "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(round(launches_per_iter * n_done)),
        "clocks": clk.summary(),
        "t_create_ms": st0["t_create_ms"], "t_generate_s": t_gen,
    }
    if args.solve:
        # time to (1+eps) solution (BASELINE metric): one full mwu_solve, all probes of the outer
        # bisection, device-timed inside the library (mwu_stats.t_solve_ms; create excluded)
        del S
        torch.cuda.empty_cache()
        S3 = Solver.graph(kind, G.src, G.dst, G.n_vertices, G.n_left if kind == "bmatch" else 0, **opts)
        S3.solve(eps)
        s3 = S3.stats()
        line["time_to_solution"] = {
            "ms": s3["t_solve_ms"], "loop_ms": s3["t_loop_ms"], "iters_total": s3["iters_total"], "probes": s3["probes"],
            "iterations_per_s": s3["iters_total"] / (s3["t_loop_ms"] / 1000.0) if s3["t_loop_ms"] > 0 else None,
            "roofline_frac_of_8TBs": (balg * s3["iters_total"] / (s3["t_loop_ms"] / 1000.0) / 8e12) if s3["t_loop_ms"] > 0 else None,
            "search_passes_per_iter": s3["search_passes"] / max(1, s3["iters_total"]),
            "objective": s3["objective"], "bound": s3["bound"], "certificate": s3["certificate"],
            "near_tie_count": s3["near_tie_count"], "t_phase_ms": s3["t_phase_ms"], "eps": eps}
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--max-iter", type=int, default=5000)
    ap.add_argument("--profile-iters", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-solve", dest="solve", action="store_false",
                    help="skip the full solve (time to (1+eps) solution), timed by default")
    ap.add_argument("--shard", action="store_true", help="sharded engine even with one rank (plumbing check)")
    ap.add_argument("--block-l", type=int, default=0, help="mwu_options.block_l (0: default L2 block shape)")
    ap.add_argument("--block-r", type=int, default=0, help="mwu_options.block_r (0: default L2 block shape)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    rc = run_ours(args)
    try:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass
    return rc


if __name__ == "__main__":
    sys.exit(main())
