# round-1 evidence: GPU tests, bench line, launch list, ncu captures of the sweep kernels
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_r01.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r01e.log 2>&1
timeout 300 python tools/prof_sweep.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01e.csv python tools/prof_sweep.py > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 9 -c 1 -o gpurun_out/prof_solve_r01e python tools/prof_sweep.py > gpurun_out/ncu_solve.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 9 -c 1 -o gpurun_out/prof_split_r01e python tools/prof_sweep.py > gpurun_out/ncu_split.log 2>&1
