#!/usr/bin/env python
"""Copy one evidence run (tools/evidence.sh outputs in gpurun_out/) into profiles/ under a round
tag: bench lines, pytest / smoke logs, the mwu:: launch-list summary, the ncu --set full summary
of the column and search kernels, and profiles/ncu_traffic.json (DRAM bytes per launch that
bench.py reports as roofline.traffic).   usage: python tools/round_profiles.py r1d"""
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

for src, dst in [("bench_default.log", f"bench_{tag}_c4.log"), ("pytest_gpu.log", f"pytest_gpu_{tag}.log"),
                 ("smoke.log", f"smoke_{tag}.log")] + [(f"bench_{w}.log", f"bench_{tag}_{w}.log") for w in ("c1", "c2", "c3", "c5")]:
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))

# launch list: mwu:: kernels of the bench command (profile_iters launches + probe init)
rows = [r for r in csv.reader(l for l in open(os.path.join(G, "launches.csv")) if l.startswith('"'))]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows[1:]:
    if r[ik].startswith("mwu::") or "mwu::" in r[ik][:12]:
        per[(r[iid], r[ik].split("(")[0])][r[im]] = float(r[iv].replace(",", ""))
with open(os.path.join(P, f"launches_c4_{tag}_mwu.csv"), "w") as f:
    w = csv.writer(f)
    w.writerow(["id", "kernel", "time_ns", "dram_read", "dram_write"])
    for (i, k), m in sorted(per.items(), key=lambda kv: int(kv[0][0])):
        w.writerow([i, k, m.get("gpu__time_duration.sum", 0), m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)])
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, k), m in per.items():
    a = agg[k]; a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0); a[3] += m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
out = [f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
       f"python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e   (B200, round 1, {tag})",
       "mwu:: kernels only (the timed steps run inside a CUDA graph with conditional nodes, which ncu does not",
       "replay; these launches are the host-driven per-phase profile_iters iterations and the probe inits).",
       "Per-launch times are cold-cache and serialised: compare shares, not absolutes.", "",
       f"{'kernel':40s} {'launches':>8s} {'time ms':>10s} {'share':>6s} {'avg ms':>8s} {'DRAM GB/launch':>14s} {'GB/s':>8s}"]
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    t_ms = a[1] / 1e6
    gb = (a[2] + a[3]) / a[0] / 1e9
    out.append(f"{k[:40]:40s} {a[0]:8d} {t_ms:10.3f} {100*a[1]/tot:5.1f}% {t_ms/a[0]:8.3f} {gb:14.3f} {gb/(t_ms/a[0]/1e3):8.0f}")
open(os.path.join(P, f"launches_c4_{tag}_summary.txt"), "w").write("\n".join(out) + "\n")
traffic = {"c4": {}}
for phase, k in (("column", "mwu::col_densest_fast"), ("search", "mwu::search_pass")):
    a = agg[k]
    traffic["c4"][phase] = {"kernel": k, "dram_bytes_per_launch": (a[2] + a[3]) / max(a[0], 1), "launches": a[0],
                            "source": f"profiles/launches_c4_{tag}_summary.txt (dram__bytes_read+write of the "
                                      "profile_iters launches of the bench command)"}
json.dump(traffic, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)

# ncu --set full summary of the captured column / search launches
rep = os.path.join(G, "prof_full.ncu-rep")
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hh = rr[0]
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
            "launch__registers_per_thread", "smsp__inst_executed.sum"]
    lines = ["ncu --set full --clock-control none --import-source on -k regex:'col_densest_fast|search_pass' -s 72 -c 2 "
             f"python tools/diag.py --iters 24 --active 0   (c4, iteration ~24 of the first probe; {tag})", ""]
    for r in rr[2:]:
        d = dict(zip(hh, r))
        lines.append(d.get("Kernel Name", "?").split("(")[0])
        for k in keys:
            if k in d:
                lines.append(f"  {k} = {d[k]}")
    open(os.path.join(P, f"ncu_full_c4_{tag}.txt"), "w").write("\n".join(lines) + "\n")
print("ok", tag)
