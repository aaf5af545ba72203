#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for b in 1 2 4; do
  echo "blocks=$b" >> gpurun_out/r02as.json
  DD_MCF_BLOCKS=$b timeout 600 python tools/flow256_probe.py >> gpurun_out/r02as.json 2>> gpurun_out/r02as.err
done
echo done
