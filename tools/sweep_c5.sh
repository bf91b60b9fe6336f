set -u
mkdir -p gpurun_out
for so in var/*.so; do
  echo "== $so" >> gpurun_out/sweep_c5.log
  MWU_SO=$PWD/$so timeout 400 python bench.py --workload c5 --steps 6 --warmup 3 --no-cpu --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print(round(j['value'],2), {k:round(v['ms_per_launch'],3) for k,v in j['phases'].items()})
" >> gpurun_out/sweep_c5.log
done
