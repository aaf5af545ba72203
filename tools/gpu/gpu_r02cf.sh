#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
DD_MS_TIMERS=1 timeout 900 python tests/diag/cfg5_ms_probe.py > gpurun_out/r02cf_touch48.jsonl 2> gpurun_out/r02cf_touch48.err
DD_POOL_RESERVE_GB=100 timeout 900 python tests/diag/cfg5_ms_probe.py > gpurun_out/r02cf_touch100.jsonl 2> gpurun_out/r02cf_touch100.err
echo done
