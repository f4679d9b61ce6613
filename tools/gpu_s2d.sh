#!/bin/bash
# Session 2, call D: N-GPU validation of the current build: multi-GPU tests + default sliced bench
# (torchrun, one rank per GPU) + the reference arm.
N=${1:-2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/s2d_multi_n$N.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/s2d_multi_n$N.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $N --steps 16 --warmup 3 > gpurun_out/s2d_bench_n$N.json 2> gpurun_out/s2d_bench_n$N.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/s2d_bench_n$N.json; grep "bench r0" gpurun_out/s2d_bench_n$N.err | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29592 bench.py --impl reference --gpus $N --steps 2 --warmup 1 > gpurun_out/s2d_ref_n$N.json 2> gpurun_out/s2d_ref_n$N.err; echo "ref rc=$?"; tail -c 400 gpurun_out/s2d_ref_n$N.json
