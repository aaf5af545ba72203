#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python tests/diag/cluster_prof.py > gpurun_out/r02ca_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sweep_kernel_cl" -c 2 \
  -o gpurun_out/r02ca_cluster python tests/diag/cluster_prof.py > gpurun_out/r02ca_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r02ca_ncu.log
echo done
