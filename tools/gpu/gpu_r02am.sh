#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_MS_TIMERS=1 LEVELS=8 REPS=6 timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02am_probe.jsonl 2>> gpurun_out/r02am.err
echo done
