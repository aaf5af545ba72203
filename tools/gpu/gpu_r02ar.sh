#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/flow256_probe.py > gpurun_out/r02ar.json 2> gpurun_out/r02ar.err
echo done
