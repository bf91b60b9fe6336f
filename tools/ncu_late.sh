#!/bin/bash
# ncu --set full of the c4 column and search kernels in a LATE iteration of the final probe
# (bound = the solve's answer, after 1500 iterations): the regime that dominates a full solve
mkdir -p gpurun_out
W=${WL:-c4}; B=${BOUND:-1162.4448479376103}; K=${SKIP:-1500}
timeout 900 python tools/diag.py --workload $W --bound $B --skip $K --iters 4 --active 1 > gpurun_out/diag_late_$W.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"col_|search_pass" -s $((K*3)) -c 3 \
    -o /tmp/prof_late python tools/diag.py --workload $W --bound $B --skip $K --iters 2 --active 0 > gpurun_out/ncu_late_$W.log 2>&1
ncu -i /tmp/prof_late.ncu-rep --page raw --csv > gpurun_out/prof_late_${W}_raw.csv 2>/dev/null
ncu -i /tmp/prof_late.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/prof_late_${W}_src.csv.gz
