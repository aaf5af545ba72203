#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02af_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02af_pytest.log
echo done
