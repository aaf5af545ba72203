mkdir -p gpurun_out
DD_LIB_PATH=tools/data/libdomdec_r01.so timeout 300 python tests/diag/debug_traj2.py cfg2_bumps > gpurun_out/r02c_debug_old.log 2>&1
