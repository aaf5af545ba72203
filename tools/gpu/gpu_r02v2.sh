#!/bin/bash
# X2 pairs: A/B of the pure sweep (previous build y.so vs new), then the sweep parity tests
mkdir -p gpurun_out
for lib in new y new y; do
  if [ $lib = y ]; then export DD_LIB_PATH=$PWD/abtmp/y.so; else unset DD_LIB_PATH; fi
  timeout 300 python tools/sweep_frac_probe.py >> gpurun_out/r02v2_ab.jsonl 2>&1
done
unset DD_LIB_PATH
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_cell_sizes.py tests/test_gpu_cluster.py tests/test_gpu_rectangular.py > gpurun_out/r02v2_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r02v2_pytest.txt
tail -3 gpurun_out/r02v2_pytest.txt
cat gpurun_out/r02v2_ab.jsonl
