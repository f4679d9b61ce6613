#!/bin/bash
# Round 2, call bb (4-GPU box): last multi-GPU regression after the router / P2P changes: all multi-GPU
# tests, default bench at N = 4 and N = 2 (GPUs 0-1).
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r2bb_multi_tests.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/r2bb_multi_tests.log
timeout 900 $TR --nproc-per-node 4 --master-port 29611 bench.py --gpus 4 > gpurun_out/r2bb_bench_n4.json 2> gpurun_out/r2bb_bench_n4.err; echo "bench n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29612 bench.py --gpus 2 > gpurun_out/r2bb_bench_n2.json 2> gpurun_out/r2bb_bench_n2.err; echo "bench n2 rc=$?"
for n in 4 2; do python - $n <<'P'
import json, sys
b = json.load(open(f"gpurun_out/r2bb_bench_n{sys.argv[1]}.json"))
print(sys.argv[1], "tok/s", round(b["value"], 3), "link", round(b["host_link"]["frac"], 3), "resident", round(b["resident"]["value"], 1),
      "router us", round(b["engine"]["us_router"], 1), "clocks", b["clocks"]["reasons"], "eq1", {k: b.get("eq1", {}).get(k) for k in ("N_G", "io_bottlenecked")})
P
done
