mkdir -p gpurun_out
start=$(date +%s)
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
echo "bench wall $(( $(date +%s) - start )) s" >> gpurun_out/r02i_bench.err
timeout 900 python -m pytest tests/test_sanitizer.py "tests/test_gpu_multiscale.py::test_multiscale_converged_parity_cfg2" -q --timeout 900 -p no:cacheprovider > gpurun_out/r02i_pytest.log 2>&1
