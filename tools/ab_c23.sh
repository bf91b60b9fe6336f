#!/bin/bash
# A/B of ab/<variant>.so on chosen workloads: "variant:wl,wl ..." pairs in $1..; bench window + full solve.
mkdir -p gpurun_out
cp paper_2307_03307_b200/libmwu.so /tmp/libmwu_keep.so
for spec in "$@"; do
  so=ab/${spec%%:*}.so; wls=${spec#*:}
  cp $so paper_2307_03307_b200/libmwu.so; touch paper_2307_03307_b200/libmwu.so
  for wl in ${wls//,/ }; do
    echo "== $so $wl" >> gpurun_out/ab_c23.log
    timeout 600 python bench.py --workload $wl --no-cpu --no-e2e --steps 20 --warmup 5 > /tmp/ab_out.txt 2>&1
    python - >> gpurun_out/ab_c23.log <<'PY'
import json
for l in open('/tmp/ab_out.txt'):
    if l.startswith('{'):
        j = json.loads(l); t = j.get('time_to_solution') or {}
        print(round(j['value'], 2), round(j['ms_per_step'], 4), {k: round(v['ms_per_iter'], 4) for k, v in j['phases'].items()},
              j['search_passes_per_iter'], 'solve', t.get('ms'), t.get('iters_total'), t.get('objective'),
              {k: round(v, 1) for k, v in (t.get('t_phase_ms') or {}).items()})
        break
else:
    print(open('/tmp/ab_out.txt').read()[-1500:])
PY
  done
done
cp /tmp/libmwu_keep.so paper_2307_03307_b200/libmwu.so
cat gpurun_out/ab_c23.log
