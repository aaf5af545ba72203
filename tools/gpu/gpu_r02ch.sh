#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_MS_TIMERS=1 timeout 900 python tests/diag/cfg5_ms_probe.py > gpurun_out/r02ch_cfg5.jsonl 2> gpurun_out/r02ch.err
LEVELS=8 REPS=3 EPS_SCALE=4 timeout 600 python tools/ms_sweep_probe.py > gpurun_out/r02ch_ms.jsonl 2>> gpurun_out/r02ch.err
timeout 1200 python -m pytest tests/test_gpu_multiscale.py tests/test_gpu_cluster.py -q -x -p no:cacheprovider > gpurun_out/r02ch_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ch_pytest.log
echo done
