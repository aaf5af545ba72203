#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_init_errors.py -q -p no:cacheprovider > gpurun_out/r02by_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02by_pytest.log
echo done
