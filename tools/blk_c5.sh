# c5 under several L2-block shapes (MWU_BLOCK_L / MWU_BLOCK_R)
set -u
mkdir -p gpurun_out
for lr in "22 20" "27 22" "27 21" "24 22"; do
  set -- $lr
  echo "== $1 $2" >> gpurun_out/blk_c5.log
  MWU_BLOCK_L=$1 MWU_BLOCK_R=$2 timeout 400 python bench.py --workload c5 --steps 6 --warmup 3 --no-cpu --no-e2e 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        j=json.loads(l); print(round(j['value'],2), {k:round(v['ms_per_launch'],3) for k,v in j['phases'].items()})
" >> gpurun_out/blk_c5.log
done
