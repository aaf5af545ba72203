mkdir -p gpurun_out
N=1024 LEVELS=6 timeout 600 python tests/diag/ms_layer_probe.py > gpurun_out/r02o_layers.jsonl 2>&1
N=1024 LEVELS=5,6 FLOW_EVERY=1 timeout 600 python tools/ms_probe.py > gpurun_out/r02o_ms1024.jsonl 2>&1
