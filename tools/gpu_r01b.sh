# round-1 evidence: GPU tests, bench line, launch list, ncu captures of the sweep kernels
DD_MCF_TIMERS=1 timeout 200 python tools/warm_check.py 1024,4,3 > gpurun_out/timers_final.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_r01g.log 2>&1
timeout 300 python tools/prof_sweep.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01g.csv python tools/prof_sweep.py > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 9 -c 1 -o gpurun_out/prof_solve_r01g python tools/prof_sweep.py > gpurun_out/ncu_solve.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 9 -c 1 -o gpurun_out/prof_split_r01g python tools/prof_sweep.py > gpurun_out/ncu_split.log 2>&1
