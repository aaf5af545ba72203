mkdir -p gpurun_out
N=1024 LEVELS=5,6 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py > gpurun_out/r02n_ms1024.jsonl 2>&1
timeout 1200 python -m pytest tests/test_gpu_multiscale.py tests/test_gpu_glued.py "tests/test_gpu_parity.py::test_first_sweep_eps_sweep_sampled" -q --timeout 900 -p no:cacheprovider > gpurun_out/r02n_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02n_pytest.log
