#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 16 32 64; do
  echo "sweeps=$k" >> gpurun_out/r02bn.jsonl
  DD_MCF_SWEEPS=$k timeout 600 python tools/flow256_probe.py >> gpurun_out/r02bn.jsonl 2>> gpurun_out/r02bn.err
done
for g in 4 16; do
  echo "gut=$g" >> gpurun_out/r02bn.jsonl
  DD_MCF_GUT=$g timeout 600 python tools/flow256_probe.py >> gpurun_out/r02bn.jsonl 2>> gpurun_out/r02bn.err
done
echo done
