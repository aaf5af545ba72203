#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
LEVELS=8 timeout 600 python tests/diag/ms_layer_probe.py > gpurun_out/r02aw_layers.jsonl 2> gpurun_out/r02aw.err
echo done
