#!/bin/bash
# Run the c4 bench (or $WL) once per ab/*.so variant (copied over the in-tree library); results in
# gpurun_out/ab.log.   tools/ab_run.sh [bench args...]
mkdir -p gpurun_out
cp paper_2307_03307_b200/libmwu.so /tmp/libmwu_keep.so
for so in ab/*.so; do
  cp $so paper_2307_03307_b200/libmwu.so
  touch paper_2307_03307_b200/libmwu.so
  echo "== $so" >> gpurun_out/ab.log
  timeout 900 python bench.py --no-cpu --no-e2e "$@" > /tmp/ab_out.txt 2>&1; tail -5 /tmp/ab_out.txt | grep -v "^{" >> gpurun_out/ab.log; cat /tmp/ab_out.txt | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print(round(j['value'],2), round(j['ms_per_step'],3), {k:round(v['ms_per_iter'],3) for k,v in j['phases'].items()}, j['search_passes_per_iter'], j.get('time_to_solution'))
" >> gpurun_out/ab.log
done
cp /tmp/libmwu_keep.so paper_2307_03307_b200/libmwu.so
