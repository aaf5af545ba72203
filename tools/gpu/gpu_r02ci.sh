#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
LEVELS=8 REPS=4 EPS_SCALE=4 STAGE_CYCLES=1 timeout 600 python tools/ms_sweep_probe.py > gpurun_out/r02ci_ms.jsonl 2>> gpurun_out/r02ci.err
echo done
