mkdir -p gpurun_out
N=1024 LEVELS=6,5,6 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py > gpurun_out/r02r_ms1024.jsonl 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiscale.py -q -x --timeout 600 -p no:cacheprovider -k "size_classes or hull_wider or multiscale_matches or refine or first_sweep_parity" > gpurun_out/r02r_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02r_pytest.log
