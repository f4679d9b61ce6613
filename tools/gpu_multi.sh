#!/bin/bash
# Multi-GPU call: box probe (RAM/topology/concurrent H2D), multi-GPU parity test, bench at N GPUs.
N=${1:-2}
mkdir -p gpurun_out
free -g > gpurun_out/probe_n$N.txt; nproc >> gpurun_out/probe_n$N.txt; nvidia-smi topo -m >> gpurun_out/probe_n$N.txt 2>&1
cat gpurun_out/probe_n$N.txt | head -20
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_tests_n$N.log 2>&1; echo "multi tests rc=$?"; tail -5 gpurun_out/multi_tests_n$N.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 8 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err; echo "bench rc=$?"
cat gpurun_out/bench_n$N.json; tail -5 gpurun_out/bench_n$N.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 tools/sweep.py --out gpurun_out/sweep_n$N.jsonl > gpurun_out/sweep_n$N.log 2>&1; echo "sweep rc=$?"
grep '^{' gpurun_out/sweep_n$N.log
