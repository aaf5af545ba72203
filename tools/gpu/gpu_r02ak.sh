#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
LEVELS=8 REPS=6 timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02ak_probe.jsonl 2>> gpurun_out/r02ak.err
echo done
