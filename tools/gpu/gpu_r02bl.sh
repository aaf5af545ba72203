#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for r in 1 2; do
for L in lib_base.so lib_noinl.so; do
  DD_LIB_PATH=$PWD/tools/data/$L timeout 600 python tools/sweep_frac_probe.py >> gpurun_out/r02bl.jsonl 2>> gpurun_out/r02bl.err
done
done
echo done
