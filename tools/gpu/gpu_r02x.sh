#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cluster.py tests/test_gpu_parity.py -k "cluster or hull_wider or size_classes" -q -x > gpurun_out/r02x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_pytest.log
for c in 0 8; do
  DD_H_CLUSTER=$c timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02x_probe.jsonl 2>> gpurun_out/r02x_probe.err
done
echo done
