mkdir -p gpurun_out
N=256 LEVELS=3 timeout 600 python tests/diag/nan_probe.py > gpurun_out/r02p_nan.log 2>&1
N=512 LEVELS=4 timeout 600 python tests/diag/nan_probe.py >> gpurun_out/r02p_nan.log 2>&1
