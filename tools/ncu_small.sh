#!/bin/bash
# ncu --set full of the c2 / c3 per-iteration kernels (search_pass, the scatters, the compaction)
# on host-driven launches (tools/diag.py, use_graph=0), plus raw / source CSV summaries in
# gpurun_out/, and the graph-launched per-phase device times of the same iterations.
mkdir -p gpurun_out
for w in c2 c3; do
  timeout 300 python tools/diag.py --workload $w --iters 12 --active 0 --phases 1 > gpurun_out/diag_$w.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k regex:"search_pass|vc_scatter|csr_scatter|edge_sum_compact|col_vertex|update_rows|inactive" -s 40 -c 8 \
      -o /tmp/prof_$w python tools/diag.py --workload $w --iters 12 --active 0 > gpurun_out/ncu_full_$w.log 2>&1
  ncu -i /tmp/prof_$w.ncu-rep --page raw --csv > gpurun_out/prof_${w}_raw.csv 2>/dev/null
  ncu -i /tmp/prof_$w.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/prof_${w}_src.csv.gz
done
