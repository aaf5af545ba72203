timeout 400 python bench.py --no-ttc --cpu-seconds 10 > gpurun_out/bench_r01b.log 2>&1
timeout 300 python tools/prof_sweep.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python tools/prof_sweep.py > gpurun_out/ncu_launch.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:solve_kernel -s 9 -c 1 -o gpurun_out/prof_solve_r01b python tools/prof_sweep.py > gpurun_out/ncu_solve.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:split_kernel -s 9 -c 1 -o gpurun_out/prof_split_r01b python tools/prof_sweep.py > gpurun_out/ncu_split.log 2>&1
DD_DEBUG_OVF=1 timeout 400 python tools/trajectory.py --N 1024 --s 4 --theta 5 --cycles 90 --seconds 380 2>&1 | grep -v "DD_DEBUG_OVF" > gpurun_out/traj_nc.log
