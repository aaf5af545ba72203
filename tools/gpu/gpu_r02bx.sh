#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
/usr/bin/time -v true 2>/dev/null; start=$(date +%s)
timeout 1500 python -m pytest tests/test_gpu_parity.py -k full_size_sampled -q -p no:cacheprovider --durations=5 > gpurun_out/r02bx_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02bx_pytest.log
echo "wall $(( $(date +%s) - start )) s" >> gpurun_out/r02bx_pytest.log
echo done
