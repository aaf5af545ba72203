#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 2 4 6; do
  echo "gut=$k" >> gpurun_out/r02bd_mcf.jsonl
  DD_MCF_GUT=$k CYCLES=8 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02bd_mcf.jsonl 2>> gpurun_out/r02bd_mcf.err
done
for r in 8 32; do
  echo "gut=4 r=$r" >> gpurun_out/r02bd_mcf.jsonl
  DD_MCF_GUT=4 DD_MCF_R=$r CYCLES=8 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02bd_mcf.jsonl 2>> gpurun_out/r02bd_mcf.err
done
echo done
