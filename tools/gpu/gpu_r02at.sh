#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_MCF_WARM=0 timeout 600 python tools/flow256_probe.py >> gpurun_out/r02at.json 2>> gpurun_out/r02at.err
echo done
