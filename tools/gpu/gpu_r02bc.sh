#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 0 10 25 50 100; do
  echo "guw=$k" >> gpurun_out/r02bc_mcf.jsonl
  DD_MCF_GUW=$k CYCLES=8 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02bc_mcf.jsonl 2>> gpurun_out/r02bc_mcf.err
done
echo done
