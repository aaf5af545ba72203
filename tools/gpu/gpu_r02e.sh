mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiscale.py "tests/test_gpu_parity.py::test_stationary_update_after_moving_flow_is_identity" "tests/test_gpu_parity.py::test_primal_dual_gap_parity" -q --timeout 600 -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02e_pytest.log
