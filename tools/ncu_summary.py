#!/usr/bin/env python
"""Summarise an ncu --csv launch list (per-kernel launches, device time, DRAM bytes, share)."""
import csv, sys, collections
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[(r[iid], r[ik].split("(")[0])][r[im]] = float(r[iv].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (i, k), m in per.items():
    a = agg[k]; a[0] += 1; a[1] += m.get("gpu__time_duration.sum", 0); a[2] += m.get("dram__bytes_read.sum", 0); a[3] += m.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'time ms':>10s} {'share':>6s} {'avg ms':>8s} {'DRAM GB/launch':>14s} {'GB/s':>8s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    t_ms = a[1] / 1e6
    gb = (a[2] + a[3]) / a[0] / 1e9
    print(f"{k[:40]:40s} {a[0]:8d} {t_ms:10.3f} {100*a[1]/tot:5.1f}% {t_ms/a[0]:8.3f} {gb:14.3f} {gb/(t_ms/a[0]/1e3):8.0f}")
