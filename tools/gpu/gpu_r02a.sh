# round 2: bench-trajectory diagnostics (hull sizes, per-sweep time) + launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
timeout 300 python tools/traj_diag.py > gpurun_out/r02a_traj.jsonl 2> gpurun_out/r02a_traj.err
CYCLES=22 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02a_launches.csv python tools/traj_diag.py > gpurun_out/r02a_ncu.log 2>&1
echo done
