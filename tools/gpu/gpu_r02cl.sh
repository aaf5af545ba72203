#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 --no-ttc --no-extra --no-cpu > gpurun_out/r02cl_torchrun.json 2> gpurun_out/r02cl_torchrun.err
echo "rc=$?" >> gpurun_out/r02cl_torchrun.err
timeout 900 python bench.py --impl reference --gpus 1 --steps 1 --warmup 0 > gpurun_out/r02cl_ref.json 2> gpurun_out/r02cl_ref.err
echo "rc=$?" >> gpurun_out/r02cl_ref.err
echo done
