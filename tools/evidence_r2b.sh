#!/bin/bash
# launch lists (hot kernels only) of the c4 / c3 / c5 bench commands + the c4 column kernel capture
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
K='col_|search_pass|update_rows|dy_finalize|edge_sum|csr_scatter|vc_scatter|inactive|step_done'
for w in c4 c3 c5; do
  timeout 600 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3 > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"$K" -c 200 --csv --log-file gpurun_out/launches_$w.csv \
      python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3 > gpurun_out/ncu_launch_$w.log 2>&1
done
timeout 300 python tools/diag.py --workload c4 --iters 12 --active 0 > gpurun_out/diag_c4b.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_densest_fast" -s 10 -c 1 \
    -o /tmp/prof_r2_c4col python tools/diag.py --workload c4 --iters 12 --active 0 > gpurun_out/ncu_full_c4col.log 2>&1
ncu -i /tmp/prof_r2_c4col.ncu-rep --page raw --csv > gpurun_out/prof_r2_c4col_raw.csv 2>/dev/null
ncu -i /tmp/prof_r2_c4col.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/prof_r2_c4col_src.csv.gz
rm -f /tmp/prof_r2_c4col.ncu-rep
du -sh gpurun_out
