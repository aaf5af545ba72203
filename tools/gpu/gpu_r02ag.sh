#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in 0 8; do
  echo "cluster=$c" >> gpurun_out/r02ag_layers.jsonl
  THETA_DEG=5 DD_H_CLUSTER=$c timeout 600 python tests/diag/ms_layer_probe.py >> gpurun_out/r02ag_layers.jsonl 2>> gpurun_out/r02ag.err
done
for c in 0 8; do
  DD_H_CLUSTER=$c timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02ag_probe.jsonl 2>> gpurun_out/r02ag.err
done
echo done
