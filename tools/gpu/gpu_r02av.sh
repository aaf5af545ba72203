#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for k in 0 1; do
  echo "scans=$k" >> gpurun_out/r02av_mcf.jsonl
  DD_MCF_SCANS=$k CYCLES=8 timeout 600 python tools/mcf_timers_probe.py >> gpurun_out/r02av_mcf.jsonl 2>> gpurun_out/r02av_mcf.err
done
timeout 600 python tools/flow256_probe.py > gpurun_out/r02av_256.json 2>> gpurun_out/r02av_mcf.err
timeout 1200 python -m pytest tests -m gpu -q -x -k "mcf or flow or hybrid or stationary or multiscale or glued or certificate" -p no:cacheprovider > gpurun_out/r02av_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02av_pytest.log
echo done
