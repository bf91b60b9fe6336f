#!/bin/bash
# GPU check (run under gpurun): build, smoke, pytest -m gpu (optionally -k), default bench line.
#   tools/gpu_check.sh "<pytest -k expr or empty>" [bench args...]
K="$1"; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
else
  timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py --no-cpu "$@" > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/bench.log
free -g > gpurun_out/host.txt; nproc >> gpurun_out/host.txt; lscpu | grep -i "model name" >> gpurun_out/host.txt
