#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02bo_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02bo_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02bo_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02bo_smoke.log
echo done
