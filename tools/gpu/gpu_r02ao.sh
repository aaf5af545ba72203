#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CYCLES=10 timeout 600 python tools/mcf_timers_probe.py > gpurun_out/r02ao_mcf.jsonl 2> gpurun_out/r02ao_mcf.err
echo done
