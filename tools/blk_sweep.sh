# bench c4 under several L2-block shapes (bench.py --block-l / --block-r = mwu_options.block_l / block_r)
set -u
mkdir -p gpurun_out
for lr in "22 20" "24 22" "24 21" "24 20" "24 19"; do
  set -- $lr
  echo "== $1 $2" >> gpurun_out/blk2.log
  timeout 300 python bench.py --block-l $1 --block-r $2 --steps 30 --warmup 5 --no-cpu --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print(round(j['value'],2), {k:round(v['ms_per_launch'],3) for k,v in j['phases'].items()})
" >> gpurun_out/blk2.log
done
