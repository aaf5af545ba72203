#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiscale.py -q -x -p no:cacheprovider > gpurun_out/r02bg_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02bg_pytest.log
start=$(date +%s)
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02bg_bench.json 2> gpurun_out/r02bg_bench.err
echo "bench wall $(( $(date +%s) - start )) s" >> gpurun_out/r02bg_bench.err
echo done
