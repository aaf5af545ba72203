#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tests/diag/slow_cells_probe.py > gpurun_out/r02w_slow.jsonl 2> gpurun_out/r02w_slow.err
echo done
