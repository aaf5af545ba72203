#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in 0 8; do
  echo "cluster=$c" >> gpurun_out/r02y_layers.jsonl
  DD_H_CLUSTER=$c timeout 600 python tests/diag/ms_layer_probe.py >> gpurun_out/r02y_layers.jsonl 2>> gpurun_out/r02y.err
done
DD_H_CLUSTER=8 DD_H_CLUSTER_KB=64 timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02y_probe.jsonl 2>> gpurun_out/r02y.err
echo done
