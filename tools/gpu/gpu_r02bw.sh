#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tests/diag/rect_probe.py > gpurun_out/r02bw.jsonl 2> gpurun_out/r02bw.err
echo done
