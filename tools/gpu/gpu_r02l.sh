mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "first_sweep or trajectory or edge_costs or size_classes or hull_wider or hybrid_parity" > gpurun_out/r02l_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02l_pytest.log
CYCLES=25 timeout 300 python tools/traj_diag.py > gpurun_out/r02l_traj.jsonl 2> gpurun_out/r02l_traj.err
CYCLES=10 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel" -s 100 -c 5 \
  -o gpurun_out/r02l_sweep python tools/prof_sweep2.py > gpurun_out/r02l_ncu_full.log 2>&1
echo done
