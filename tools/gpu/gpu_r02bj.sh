#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python tests/diag/s8_debug.py > gpurun_out/r02bj.jsonl 2> gpurun_out/r02bj.err
echo done
