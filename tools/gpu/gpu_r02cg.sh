#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python tests/diag/soak_1024.py > gpurun_out/r02cg_soak.jsonl 2> gpurun_out/r02cg.err
echo "rc=$?" >> gpurun_out/r02cg.err
echo done
