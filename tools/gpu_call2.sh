#!/bin/bash
# A/B of the packed record streams (ab/base.so vs ab/new.so) on c2, c3, c4, then the GPU parity
# tests of the covering kinds and the c2 / c3 ncu captures with ab/new.so.
mkdir -p gpurun_out
WLS="c2 c3 c4" bash tools/ab_small.sh
cp ab/new.so paper_2307_03307_b200/libmwu.so; touch paper_2307_03307_b200/libmwu.so
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -k "vcover or domset or compact or densest" -x > gpurun_out/pytest_new.log 2>&1; echo pytest=$? >> gpurun_out/pytest_new.log
bash tools/ncu_small.sh
