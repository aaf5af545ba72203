#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tools/flow256_probe.py > gpurun_out/r02br_256.json 2> gpurun_out/r02br.err
timeout 1500 python -m pytest tests -m gpu -q -x -k "mcf or flow or hybrid or stationary or multiscale or glued or certificate or run_cycles or resume or stripe" -p no:cacheprovider > gpurun_out/r02br_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02br_pytest.log
echo done
