#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 4 8 16; do
  echo "sweeps=$k" >> gpurun_out/r02au_mcf.jsonl
  DD_MCF_SWEEPS=$k CYCLES=6 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02au_mcf.jsonl 2>> gpurun_out/r02au_mcf.err
done
echo done
