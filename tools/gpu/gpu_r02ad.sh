#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/cluster_floor_probe.py > gpurun_out/r02ad_floor.jsonl 2> gpurun_out/r02ad.err
for c in 0 8; do
  DD_H_CLUSTER=$c timeout 600 python tools/ms_sweep_probe.py >> gpurun_out/r02ad_probe.jsonl 2>> gpurun_out/r02ad.err
done
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/r02ad_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ad_pytest.log
echo done
