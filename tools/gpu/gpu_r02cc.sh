#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for L in lib_base.so lib_unroll.so; do
  DD_LIB_PATH=$PWD/tools/data/$L timeout 600 python tests/diag/cluster_time.py >> gpurun_out/r02cc.jsonl 2>> gpurun_out/r02cc.err
done
DD_LIB_PATH=$PWD/tools/data/lib_unroll.so timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -k "cluster or hull_wider or size_classes" -q -p no:cacheprovider > gpurun_out/r02cc_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02cc_pytest.log
echo done
