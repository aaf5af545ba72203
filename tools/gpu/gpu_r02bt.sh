#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CYCLES=3 timeout 300 python tools/mcf_timers_probe.py > gpurun_out/r02bt_plain.log 2>&1 &&
CYCLES=3 timeout 600 ncu --nvtx --nvtx-include "dd:flow_update/dd:min-cost flow/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02bt_nvtx.csv python tools/mcf_timers_probe.py > gpurun_out/r02bt_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02bt_ncu.log
echo done
