#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=256 CYCLES=3 timeout 900 python tools/mcf_eps_probe.py > gpurun_out/r02bk_eps.jsonl 2> gpurun_out/r02bk.err
DD_MCF_TIMERS=1 timeout 600 python tools/flow256_probe.py > gpurun_out/r02bk_256.json 2>> gpurun_out/r02bk.err
echo done
