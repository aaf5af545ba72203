#!/bin/bash
# run_cycles (CUDA-graph hybrid cycles): parity with the eager sequence, A/B timing
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_run_cycles.py -q -x > gpurun_out/r02u_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_pytest.log
true
echo done
