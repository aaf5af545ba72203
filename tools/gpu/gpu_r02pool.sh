#!/bin/bash
mkdir -p gpurun_out
for gb in 48 96 0; do
  DD_POOL_RESERVE_GB=$gb timeout 600 python tools/cfg5_ms_probe.py >> gpurun_out/r02pool.jsonl 2>&1
done
DD_MS_TIMERS=1 DD_POOL_RESERVE_GB=48 REPS=3 timeout 600 python tools/cfg5_ms_probe.py > gpurun_out/r02pool_timers.txt 2>&1
cat gpurun_out/r02pool.jsonl
