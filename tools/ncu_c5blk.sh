#!/bin/bash
# L2 / DRAM counters of the c5 column kernel at several destination block shapes
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_red.sum,lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcunit_ltcfabric_lookup_hit.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sectors_srcunit_tex_op_write.sum
for br in 20 21 22 23; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:"col_match_fast" -s 5 -c 1 --csv \
    python tools/diag.py --workload c5 --iters 7 --active 0 --block-r $br > gpurun_out/ncu_blk_$br.csv 2>&1
done
