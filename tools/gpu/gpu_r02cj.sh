#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_H_CLUSTER=8 timeout 900 python tests/diag/relerr_probe.py > gpurun_out/r02cj_relerr.jsonl 2> gpurun_out/r02cj.err
LEVELS=8 REPS=3 EPS_SCALE=4 STAGE_CYCLES=1 timeout 600 python tools/ms_sweep_probe.py > gpurun_out/r02cj_ms.jsonl 2>> gpurun_out/r02cj.err
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02cj_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02cj_pytest.log
echo done
