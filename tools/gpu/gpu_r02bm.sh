#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/sweep_frac_probe.py >> gpurun_out/r02bm.jsonl 2>> gpurun_out/r02bm.err
for m in 1 2; do
  echo "M=$m" >> gpurun_out/r02bm.jsonl
  DD_CLASS_OCC_1=$m timeout 600 python tools/sweep_frac_probe.py >> gpurun_out/r02bm.jsonl 2>> gpurun_out/r02bm.err
done
echo "S=6" >> gpurun_out/r02bm.jsonl
DD_CLASS_OCC_0=6 timeout 600 python tools/sweep_frac_probe.py >> gpurun_out/r02bm.jsonl 2>> gpurun_out/r02bm.err
echo done
