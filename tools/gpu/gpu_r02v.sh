#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for th in 1 0.5 0; do
  DD_TOL_THETA=$th timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02v_theta.jsonl 2>> gpurun_out/r02v_theta.err
done
echo done
