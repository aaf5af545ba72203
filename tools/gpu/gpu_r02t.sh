mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02t_bench.json 2> gpurun_out/r02t_bench.err
echo "bench wall $(( $(date +%s) - start )) s" >> gpurun_out/r02t_bench.err
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02t_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_pytest.log
