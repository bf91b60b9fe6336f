#!/usr/bin/env python
"""Histogram of SASS opcodes (instructions executed, stall samples) of one kernel in an ncu report."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source=sass"], capture_output=True, text=True).stdout.splitlines()
i = next(k for k, l in enumerate(out) if l.startswith('"Address"'))
rows = list(csv.reader(out[i:]))
h = rows[0]
ci, cs, cx = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
inst, stall = collections.Counter(), collections.Counter()
tot_i = tot_s = 0
for r in rows[1:]:
    if len(r) <= ci or not r[ci].strip().isdigit():
        continue
    op = r[cx].split()[0] if r[cx].split() else "?"
    if op.startswith("@"):
        op = r[cx].split()[1]
    op = op.split(".")[0]
    inst[op] += int(r[ci]); stall[op] += int(r[cs] or 0)
    tot_i += int(r[ci]); tot_s += int(r[cs] or 0)
print(f"total warp-instructions {tot_i:,}  stall samples {tot_s:,}")
for op, n in inst.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"{op:10s} {n:>14,} {100*n/tot_i:5.1f}%   stalls {100*stall[op]/max(1,tot_s):5.1f}%")
