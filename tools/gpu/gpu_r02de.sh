#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02de_bench.json 2> gpurun_out/r02de_bench.err
echo "bench wall $(( $(date +%s) - start )) s" >> gpurun_out/r02de_bench.err
timeout 2700 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02de_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02de_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02de_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r02de_smoke.log
echo done
