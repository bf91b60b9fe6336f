#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun): bench lines for c1-c5 (c4 = the default line with
# CPU baseline, e2e and the full solve), the ncu launch list of each bench command, and ncu --set full
# captures of the top kernels of c4, c5, c2, c3.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
for w in c1 c2 c3; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log
done
timeout 1500 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for w in c4 c2 c3 c5; do
  timeout 600 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3 > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"col_|search_pass|update_rows|dy_finalize|edge_sum|csr_scatter|vc_scatter|inactive|step_done" -c 200 --csv --log-file gpurun_out/launches_$w.csv \
      python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3 > gpurun_out/ncu_launch_$w.log 2>&1
done
for spec in "c4 col_densest_fast|search_pass 40" "c5 col_match_fast|search_pass 30" "c2 vc_scatter|edge_sum_compact|search_pass|col_vertex 60" "c3 csr_scatter|edge_sum_compact|search_pass|col_vertex 60"; do
  set -- $spec
  timeout 300 python tools/diag.py --workload $1 --iters 12 --active 0 > gpurun_out/diag_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c 3 \
      -o /tmp/prof_r2_$1 python tools/diag.py --workload $1 --iters 12 --active 0 > gpurun_out/ncu_full_$1.log 2>&1
  # keep the summaries only (gpurun brings back <= 64 MiB): raw metrics and per-line CUDA source stalls
  ncu -i /tmp/prof_r2_$1.ncu-rep --page raw --csv > gpurun_out/prof_r2_$1_raw.csv 2>/dev/null
  ncu -i /tmp/prof_r2_$1.ncu-rep --page source --csv --print-source cuda,sass --launch-count 1 2>/dev/null | gzip > gpurun_out/prof_r2_$1_src.csv.gz
  rm -f /tmp/prof_r2_$1.ncu-rep
done
du -sh gpurun_out
echo done
