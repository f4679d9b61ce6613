#!/bin/bash
# Round 2, call x (4-GPU box): fused P2P send ({value, epoch} pairs) as the default: all multi-GPU tests,
# default bench at N = 4 and N = 2, A/B against the separate send kernel at N = 4.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r2x_multi_tests.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/r2x_multi_tests.log
timeout 900 $TR --nproc-per-node 4 --master-port 29561 bench.py --gpus 4 > gpurun_out/r2x_bench_n4.json 2> gpurun_out/r2x_bench_n4.err; echo "bench n4 rc=$?"
ODMOE_P2P_FUSED=0 timeout 900 $TR --nproc-per-node 4 --master-port 29562 bench.py --gpus 4 --steps 10 --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 > gpurun_out/r2x_bench_n4_f0.json 2> gpurun_out/r2x_bench_n4_f0.err; echo "bench n4 f0 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29563 bench.py --gpus 2 > gpurun_out/r2x_bench_n2.json 2> gpurun_out/r2x_bench_n2.err; echo "bench n2 rc=$?"
for f in r2x_bench_n4 r2x_bench_n4_f0 r2x_bench_n2; do python - $f <<'P'
import json, sys
b = json.load(open(f"gpurun_out/{sys.argv[1]}.json"))
print(sys.argv[1], "tok/s", round(b["value"], 3), "link", round(b["host_link"]["frac"], 3), "us/expert", [round(x, 1) for x in b["roofline"]["us_per_expert_by_rank"]],
      "resident", round(b["resident"]["value"], 1), "clocks", b["clocks"]["reasons"])
P
done
