#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CYCLES=4 timeout 300 python tools/mcf_timers_probe.py > gpurun_out/r02ap_plain.log 2>&1 &&
CYCLES=4 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:mcf_kernel -s 3 -c 1 -o gpurun_out/r02ap_mcf python tools/mcf_timers_probe.py > gpurun_out/r02ap_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02ap_ncu.log
