#!/bin/bash
# Quick GPU check: build, smoke, a pytest selection, c4 bench (no CPU baseline).  Usage:
#   tools/gpu_quick.sh "<pytest -k expr or empty>" [bench args...]
K="$1"; shift
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$K" > gpurun_out/pytest_sel.log 2>&1; echo pytest=$? >> gpurun_out/pytest_sel.log
fi
timeout 600 python bench.py --no-cpu "$@" > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
