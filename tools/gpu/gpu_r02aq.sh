#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 0 4 8 16; do
  echo "async=$k" >> gpurun_out/r02aq_mcf.jsonl
  DD_MCF_ASYNC=$k CYCLES=8 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02aq_mcf.jsonl 2>> gpurun_out/r02aq_mcf.err
done
timeout 1200 python -m pytest tests -m gpu -q -x -k "mcf or flow or hybrid or stationary or multiscale or glued or stripe" -p no:cacheprovider > gpurun_out/r02aq_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02aq_pytest.log
echo done
