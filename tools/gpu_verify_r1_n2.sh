#!/bin/bash
# Re-entry verification at N (default 2): multi-GPU tests and the driver's default torchrun bench line.
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_verify_n$N.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/multi_verify_n$N.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29591 bench.py --gpus $N --steps 16 --warmup 3 > gpurun_out/bench_verify_n$N.json 2> gpurun_out/bench_verify_n$N.err; echo "bench rc=$?"; cat gpurun_out/bench_verify_n$N.json; tail -2 gpurun_out/bench_verify_n$N.err
