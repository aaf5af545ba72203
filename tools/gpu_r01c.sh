# round-1 final evidence at the last build: GPU tests, bench line, launch list, ncu captures
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r01h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r01h.log
timeout 900 python bench.py > gpurun_out/bench_r01h.log 2>&1
timeout 300 python tools/prof_sweep.py > gpurun_out/prof_plain_h.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01h.csv python tools/prof_sweep.py > gpurun_out/ncu_launch_h.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 9 -c 1 -o gpurun_out/prof_solve_r01h python tools/prof_sweep.py > gpurun_out/ncu_solve_h.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 9 -c 1 -o gpurun_out/prof_split_r01h python tools/prof_sweep.py > gpurun_out/ncu_split_h.log 2>&1
