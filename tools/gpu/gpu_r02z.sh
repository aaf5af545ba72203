#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_H_CLUSTER=8 timeout 600 python tests/diag/slow_cells_probe.py > gpurun_out/r02z_slow.jsonl 2> gpurun_out/r02z.err
echo done
