#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for L in 6 7 8; do
  LEVELS=$L timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02ah_probe.jsonl 2>> gpurun_out/r02ah.err
done
echo done
