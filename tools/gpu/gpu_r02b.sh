# round 2: fused size-class sweep -- GPU tests + trajectory timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
timeout 300 python tools/traj_diag.py > gpurun_out/r02b_traj.jsonl 2> gpurun_out/r02b_traj.err
echo done
