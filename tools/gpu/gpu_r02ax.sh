#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for m in 2000 1000 500 250; do
  MAX_ITER=$m LEVELS=8 REPS=3 timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02ax_probe.jsonl 2>> gpurun_out/r02ax.err
done
echo done
