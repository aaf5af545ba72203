#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in 1 2; do
for L in lib_base.so lib_occ8.so; do
  DD_LIB_PATH=$PWD/tools/data/$L timeout 600 python tools/sweep_frac_probe.py >> gpurun_out/r02bp.jsonl 2>> gpurun_out/r02bp.err
done
done
echo done
