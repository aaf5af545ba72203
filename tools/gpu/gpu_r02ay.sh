#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for L in lib_base.so lib_s2w32.so; do
  DD_LIB_PATH=$PWD/tools/data/$L timeout 600 python tools/sweep_frac_probe.py >> gpurun_out/r02ay.jsonl 2>> gpurun_out/r02ay.err
done
echo done
