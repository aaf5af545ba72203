#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_LIB_PATH=$PWD/tools/data/libdomdec_head.so timeout 900 python tests/diag/relerr_probe.py >> gpurun_out/r02ae.jsonl 2>> gpurun_out/r02ae.err
DD_H_CLUSTER=0 timeout 900 python tests/diag/relerr_probe.py >> gpurun_out/r02ae.jsonl 2>> gpurun_out/r02ae.err
DD_H_CLUSTER=8 timeout 900 python tests/diag/relerr_probe.py >> gpurun_out/r02ae.jsonl 2>> gpurun_out/r02ae.err
echo done
