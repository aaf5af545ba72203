#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 2 --warmup 1 --no-ttc --no-extra --no-cpu > gpurun_out/r02df_plain.json 2> gpurun_out/r02df_plain.err &&
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02df_launches.csv python bench.py --steps 2 --warmup 1 --no-ttc --no-extra --no-cpu > gpurun_out/r02df_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02df_ncu.log
echo done
