#!/bin/bash
# ncu --set full of one c5 col_match_fast launch (+ raw / source CSV summaries into gpurun_out/)
mkdir -p gpurun_out
timeout 300 python tools/diag.py --workload c5 --iters 8 --active 0 > gpurun_out/diag_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"col_match_" -s 5 -c 1 \
    -o /tmp/prof_c5col python tools/diag.py --workload c5 --iters 8 --active 0 > gpurun_out/ncu_full_c5col.log 2>&1
ncu -i /tmp/prof_c5col.ncu-rep --page raw --csv > gpurun_out/prof_c5col_raw.csv 2>/dev/null
ncu -i /tmp/prof_c5col.ncu-rep --page details --csv > gpurun_out/prof_c5col_details.csv 2>/dev/null
ncu -i /tmp/prof_c5col.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/prof_c5col_src.csv.gz
