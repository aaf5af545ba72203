#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CYCLES=4 timeout 900 python tools/mcf_eps_probe.py > gpurun_out/r02ba_eps.jsonl 2> gpurun_out/r02ba.err
for k in 1 16; do
  echo "epsmin=$k" >> gpurun_out/r02ba_warm.jsonl
  DD_MCF_EPSMIN=$k CYCLES=8 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02ba_warm.jsonl 2>> gpurun_out/r02ba.err
done
echo done
