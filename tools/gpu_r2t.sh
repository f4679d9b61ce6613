#!/bin/bash
# Round 2, call t (4-GPU box): end-of-round multi-GPU verification with the current defaults: every
# multi-GPU test (N = 2 and 4), default bench + reference arm at N = 4 and at N = 2 (GPUs 0-1).
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 2400 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/r2t_multi_tests.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/r2t_multi_tests.log
timeout 900 $TR --nproc-per-node 4 --master-port 29531 bench.py --gpus 4 > gpurun_out/r2t_bench_n4.json 2> gpurun_out/r2t_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29532 bench.py --impl reference --gpus 4 > gpurun_out/r2t_ref_n4.json 2> gpurun_out/r2t_ref_n4.err; echo "ref n4 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29533 bench.py --gpus 2 > gpurun_out/r2t_bench_n2.json 2> gpurun_out/r2t_bench_n2.err; echo "bench n2 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29534 bench.py --impl reference --gpus 2 > gpurun_out/r2t_ref_n2.json 2> gpurun_out/r2t_ref_n2.err; echo "ref n2 rc=$?"
for n in 4 2; do python - $n <<'P'
import json, sys
n = sys.argv[1]
b = json.load(open(f"gpurun_out/r2t_bench_n{n}.json"))
r = json.load(open(f"gpurun_out/r2t_ref_n{n}.json"))
print(n, "value", round(b["value"], 3), "link frac", round(b["host_link"]["frac"], 3), "resident", round(b["resident"]["value"], 1),
      "roof frac", round(b["roofline"]["frac"], 3), "clocks", b["clocks"]["reasons"], "ref", r.get("value"))
P
done
