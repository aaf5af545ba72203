# ncu evidence at the bench trajectory (cycle 10): launch list + full captures of one A and one B sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CYCLES=10 timeout 300 python tools/prof_sweep2.py > gpurun_out/r02az_plain.log 2>&1
CYCLES=10 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02az_launches.csv python tools/prof_sweep2.py > gpurun_out/r02az_ncu_launch.log 2>&1
CYCLES=10 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|k_bin" -s 120 -c 12 \
  -o gpurun_out/r02az_sweep python tools/prof_sweep2.py > gpurun_out/r02az_ncu_full.log 2>&1
echo done
