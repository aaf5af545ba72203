#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py -q -p no:cacheprovider -k stale > gpurun_out/r02cm_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02cm_pytest.log
echo done
