mkdir -p gpurun_out
nproc > gpurun_out/r02h_nproc.txt; lscpu | grep "Model name" >> gpurun_out/r02h_nproc.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
/usr/bin/time -v timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err
