mkdir -p gpurun_out
N=1024 LEVELS=5,6,4 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py > gpurun_out/r02g_ms1024.jsonl 2>&1
N=1024 THETA=5 LEVELS=5 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py >> gpurun_out/r02g_ms1024.jsonl 2>&1
