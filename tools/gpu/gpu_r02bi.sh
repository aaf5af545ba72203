#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for L in libdomdec_head.so libdomdec_r01.so; do
  echo "== $L" >> gpurun_out/r02bi_pytest.log
  DD_LIB_PATH=$PWD/tools/data/$L timeout 900 python -m pytest tests/test_gpu_cell_sizes.py -q -k "s8 and 0-" -p no:cacheprovider >> gpurun_out/r02bi_pytest.log 2>&1
done
echo done
