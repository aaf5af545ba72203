mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multiscale.py -q --timeout 600 -p no:cacheprovider > gpurun_out/r02f_pytest.log 2>&1
N=256 LEVELS=3,4 FLOW_EVERY=1,0 timeout 300 python tools/ms_probe.py > gpurun_out/r02f_ms256.jsonl 2>&1
N=1024 LEVELS=5,6 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py > gpurun_out/r02f_ms1024.jsonl 2>&1
