#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for f in 1 2 4; do
  EPS_SCALE=$f LEVELS=8 REPS=3 timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02be_probe.jsonl 2>> gpurun_out/r02be.err
done
timeout 900 python -m pytest tests/test_gpu_multiscale.py tests/test_gpu_run_cycles.py -q -x -p no:cacheprovider > gpurun_out/r02be_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02be_pytest.log
echo done
