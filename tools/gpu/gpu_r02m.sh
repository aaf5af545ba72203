mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "first_sweep or trajectory or size_classes or hull_wider or hybrid_parity" > gpurun_out/r02m_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02m_pytest.log
CYCLES=25 timeout 300 python tools/traj_diag.py > gpurun_out/r02m_traj.jsonl 2> gpurun_out/r02m_traj.err
echo done
