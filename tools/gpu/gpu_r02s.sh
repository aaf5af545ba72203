mkdir -p gpurun_out
N=1024 LEVELS=5,6,5 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py > gpurun_out/r02s_ms1024.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02s_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02s_pytest.log
CYCLES=12 timeout 1200 python tools/mcf_knobs.py > gpurun_out/r02s_knobs.jsonl 2>&1
