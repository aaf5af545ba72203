mkdir -p gpurun_out
N=256 LEVELS=3 timeout 600 python tests/diag/nan_probe.py > gpurun_out/r02q_nan.log 2>&1
N=1024 LEVELS=6 timeout 600 python tests/diag/slow_probe.py > gpurun_out/r02q_slow.jsonl 2>&1
