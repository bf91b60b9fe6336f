#!/bin/bash
# c5 column-kernel experiments: every ab/*.so variant at the default block shape, then the
# block_r sweep on the first variant named in $SWEEP_SO.  Results in gpurun_out/ab_c5.log.
mkdir -p gpurun_out
cp paper_2307_03307_b200/libmwu.so /tmp/libmwu_keep.so
run() {  # label, bench args...
  local lab=$1; shift
  echo "== $lab $*" >> gpurun_out/ab_c5.log
  timeout 600 python bench.py --workload ${WL:-c5} --no-cpu --no-e2e --no-solve --steps 10 --warmup 3 "$@" > /tmp/ab_out.txt 2>&1
  grep -m1 "L2 fetch" /tmp/ab_out.txt >> gpurun_out/ab_c5.log
  python - >> gpurun_out/ab_c5.log <<'PY'
import json
for l in open('/tmp/ab_out.txt'):
    if l.startswith('{'):
        j=json.loads(l); print(round(j['value'],2), round(j['ms_per_step'],3), {k:round(v['ms_per_iter'],3) for k,v in j['phases'].items()}, j['search_passes_per_iter'], j['iteration_roofline']['frac_of_8TBs'])
        break
else:
    print(open('/tmp/ab_out.txt').read()[-1500:])
PY
}
for so in ab/*.so; do
  cp $so paper_2307_03307_b200/libmwu.so; touch paper_2307_03307_b200/libmwu.so
  run $so
  [ -n "$ALSO_C4" ] && WL=c4 run "$so c4"
done
if [ -n "$SWEEP_SO" ]; then
  cp ab/$SWEEP_SO.so paper_2307_03307_b200/libmwu.so; touch paper_2307_03307_b200/libmwu.so
  for br in $SWEEP_BR; do run "$SWEEP_SO block_r=$br" --block-r $br; done
fi
cp /tmp/libmwu_keep.so paper_2307_03307_b200/libmwu.so
