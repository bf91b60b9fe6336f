#!/bin/bash
# Final round-2 evidence on one B200 (under gpurun), ordered so the judged items come first:
# smoke, default bench line (c4: CPU baseline, e2e, full solve), c1-c3 bench lines, reference arm,
# every GPU test, ncu launch lists + ncu --set full summaries (c4, c2, c3), then the c5 bench line.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_c4.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c4.log
for w in c1 c2 c3; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu > gpurun_out/bench_$w.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$w.log
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_ref.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for w in c4 c2 c3; do
  timeout 600 python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3 > gpurun_out/plain_$w.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"col_|search_pass|update_rows|dy_finalize|edge_sum|csr_scatter|vc_scatter|inactive|step_done" -c 200 --csv --log-file gpurun_out/launches_$w.csv \
      python bench.py --workload $w --steps 4 --warmup 3 --no-cpu --no-e2e --no-solve --profile-iters 3 > gpurun_out/ncu_launch_$w.log 2>&1
done
# ncu --set full: c4 as before; c2 after 16 matching launches (iterations 3-4); c3's first probe at
# the diag bound ends after one iteration, so its capture starts at the third matching launch
for spec in "c4 col_densest_fast|search_pass 40 3" "c2 vc_scatter|edge_sum_compact|search_pass|col_vertex|update_rows 16 8" "c3 csr_scatter|edge_sum_compact|search_pass|col_vertex|update_rows 2 8"; do
  set -- $spec
  timeout 300 python tools/diag.py --workload $1 --iters 12 --active 0 > gpurun_out/diag_$1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s $3 -c $4 \
      -o /tmp/prof_r2_$1 python tools/diag.py --workload $1 --iters 12 --active 0 > gpurun_out/ncu_full_$1.log 2>&1
  ncu -i /tmp/prof_r2_$1.ncu-rep --page raw --csv > gpurun_out/prof_r2_$1_raw.csv 2>/dev/null
  rm -f /tmp/prof_r2_$1.ncu-rep
done
timeout 1200 python bench.py --workload c5 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_c5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5.log
du -sh gpurun_out
echo done
