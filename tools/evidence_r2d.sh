#!/bin/bash
# Full round-2 evidence on one B200 (under gpurun): smoke, every GPU test, then tools/evidence_r2.sh
# (bench lines c1-c5, ncu launch lists, ncu --set full captures).  Outputs in gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$? >> gpurun_out/pytest_gpu.log
bash tools/evidence_r2.sh > gpurun_out/evidence.log 2>&1
