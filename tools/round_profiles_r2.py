#!/usr/bin/env python
"""Summarise a tools/evidence_r2.sh run (gpurun_out/) into profiles/: bench lines, the mwu:: launch
list of each workload's bench command (per-kernel share, DRAM bytes per launch), the ncu --set full
metrics of the captured top kernels, and profiles/ncu_traffic.json (the per-phase DRAM bytes bench.py
prints beside its algorithmic credits).   usage: python tools/round_profiles_r2.py r2a"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
tag = sys.argv[1]
PHASE_OF = {"col_densest_fast": "column", "inactive_exact": "column", "col_match_fast": "column",
            "vc_scatter": "column", "csr_scatter": "column", "col_vertex": "column",
            "dy_finalize": "step", "edge_sum_compact": "step", "inactive_exact_dz": "step", "step_done": "step",
            "search_pass": "search", "update_rows": "update"}

for w in ("c1", "c2", "c3", "c4", "c5"):
    src = os.path.join(G, f"bench_{w}.log")
    if os.path.exists(src):
        shutil.copy(src, os.path.join(P, f"bench_{tag}_{w}.log"))
for f in ("pytest_gpu.log", "smoke.log"):
    if os.path.exists(os.path.join(G, f)):
        shutil.copy(os.path.join(G, f), os.path.join(P, f.replace(".log", f"_{tag}.log")))

traffic = {}
for w in ("c4", "c2", "c3", "c5"):
    path = os.path.join(G, f"launches_{w}.csv")
    if not os.path.exists(path):
        continue
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        name = r[ik].split("(")[0].replace("void ", "").replace("mwu::", "")
        if name in PHASE_OF or name.startswith(("col_", "search", "update", "dy_", "edge_", "csr_", "vc_", "inactive")):
            per[(r[iid], "mwu::" + name)][r[im]] = float(r[iv].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (i, k), m in per.items():
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0)
        a[2] += m.get("dram__bytes_read.sum", 0)
        a[3] += m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values()) or 1.0
    out = [f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 300 "
           f"python bench.py --workload {w} --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3   "
           f"(B200, round 2, {tag})",
           "mwu:: kernels only: the timed steps run inside a CUDA graph (conditional nodes), which ncu does not",
           "replay; these launches are the host-driven per-phase profile_iters iterations and the probe inits.",
           "Per-launch times are cold-cache and serialised: compare shares, not absolutes.", "",
           f"{'kernel':40s} {'launches':>8s} {'time ms':>10s} {'share':>6s} {'avg ms':>8s} {'DRAM GB/launch':>14s} {'GB/s':>8s}"]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        t_ms = a[1] / 1e6
        gb = (a[2] + a[3]) / a[0] / 1e9
        out.append(f"{k[:40]:40s} {a[0]:8d} {t_ms:10.3f} {100 * a[1] / tot:5.1f}% {t_ms / a[0]:8.3f} {gb:14.3f} "
                   f"{gb / max(t_ms / a[0] / 1e3, 1e-12):8.0f}")
    open(os.path.join(P, f"launches_{w}_{tag}_summary.txt"), "w").write("\n".join(out) + "\n")
    ph = collections.defaultdict(lambda: [0.0, 0])
    for k, a in agg.items():
        name = k.replace("mwu::", "")
        if name in PHASE_OF:
            p = PHASE_OF[name]
            ph[p][0] += a[2] + a[3]
            ph[p][1] = max(ph[p][1], a[0])
    traffic[w] = {p: {"dram_bytes_per_launch": v[0] / max(v[1], 1), "launches": v[1],
                      "source": f"profiles/launches_{w}_{tag}_summary.txt (dram__bytes_read+write per launch of the "
                                "phase's kernels, profile_iters launches of the bench command)"}
                  for p, v in ph.items()}
if traffic:
    json.dump(traffic, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)

keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum"]
for w in ("c4", "c5", "c2", "c3"):
    rawp = os.path.join(G, f"prof_r2_{w}_raw.csv")
    if not os.path.exists(rawp):
        continue
    rr = list(csv.reader(open(rawp)))
    if not rr:
        continue
    hh = rr[0]
    skip = {"c4": "-s 40 -c 3", "c2": "-s 16 -c 8", "c3": "-s 2 -c 8", "c5": "-s 30 -c 3"}[w]
    lines = [f"ncu --set full --clock-control none --import-source on {skip} (tools/evidence_r2f.sh; -s/-c of earlier "
             f"tags: tools/evidence_r2.sh) python tools/diag.py --workload {w} --iters 12 --active 0   "
             f"({w}, first probe, host-driven iterations; round 2, {tag})", ""]
    for r in rr[2:]:
        d = dict(zip(hh, r))
        lines.append(d.get("Kernel Name", "?").split("(")[0])
        for k in keys:
            if k in d:
                lines.append(f"  {k} = {d[k]}")
    open(os.path.join(P, f"ncu_full_{w}_{tag}.txt"), "w").write("\n".join(lines) + "\n")
print("ok", tag, sorted(traffic))
