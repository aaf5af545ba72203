# ncu of one A sweep at the bench trajectory (cycle 10) after the Y/X2 trims
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CYCLES=10 timeout 300 python tools/prof_sweep2.py > gpurun_out/r02db_plain.log 2>&1 && \
CYCLES=10 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel|k_bin" -s 120 -c 6 \
  -o gpurun_out/r02db_sweep python tools/prof_sweep2.py > gpurun_out/r02db_ncu_full.log 2>&1
echo done
