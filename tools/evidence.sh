#!/bin/bash
# Round evidence on one B200 (run under gpurun): smoke, full GPU tests, the default bench line,
# the other configs' bench lines, the ncu launch list of the default bench command, and one
# ncu --set full capture of the dominant kernels (column + search) of c4.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
for w in c1 c2 c3 c5; do
  timeout 600 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$w.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$w.log
done
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_launches.log 2>&1
timeout 200 python tools/diag.py --iters 24 --active 0 > gpurun_out/diag_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_densest_fast|search_pass" -s 72 -c 2 \
    -o gpurun_out/prof_full python tools/diag.py --iters 24 --active 0 > gpurun_out/ncu_full.log 2>&1
echo done
