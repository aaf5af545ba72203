#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in 1 2; do
for f in 2 4; do
  echo "stagecap=$c" >> gpurun_out/r02bf_probe.jsonl
  DD_MS_STAGE_CYCLES=$c EPS_SCALE=$f LEVELS=8 REPS=2 timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02bf_probe.jsonl 2>> gpurun_out/r02bf.err
done
done
echo done
