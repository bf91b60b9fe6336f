#!/bin/bash
# c4 column experiments: each ab/*.so on the bench window (iterations 6-15 of the first probe) and
# on late iterations of the final probe (host-driven per-phase times).  gpurun_out/ab_c4.log
mkdir -p gpurun_out
cp paper_2307_03307_b200/libmwu.so /tmp/libmwu_keep.so
for so in ab/*.so; do
  cp $so paper_2307_03307_b200/libmwu.so; touch paper_2307_03307_b200/libmwu.so
  echo "== $so" >> gpurun_out/ab_c4.log
  timeout 600 python bench.py --workload c4 --no-cpu --no-e2e --no-solve --steps 10 --warmup 3 > /tmp/ab_out.txt 2>&1
  python - >> gpurun_out/ab_c4.log <<'PY'
import json
for l in open('/tmp/ab_out.txt'):
    if l.startswith('{'):
        j=json.loads(l); print(round(j['value'],2), round(j['ms_per_step'],3), {k:round(v['ms_per_iter'],3) for k,v in j['phases'].items()}, j['search_passes_per_iter'], j['iteration_roofline']['frac_of_8TBs']); break
else: print(open('/tmp/ab_out.txt').read()[-1500:])
PY
  timeout 600 python tools/diag.py --workload c4 --bound 1162.4448479376103 --skip 1500 --iters 6 --active 0 --phases 1 2>&1 | tail -4 >> gpurun_out/ab_c4.log
done
cp /tmp/libmwu_keep.so paper_2307_03307_b200/libmwu.so
