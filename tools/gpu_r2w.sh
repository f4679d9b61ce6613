#!/bin/bash
# Round 2, call w (2-GPU box): P2P combine in the LL format ({value, epoch} pairs, no fence / flag):
# multi-GPU tests (incl. the fused send, bitwise), then the A/B fused send vs separate send kernel at N = 2.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -x -k emulation > gpurun_out/r2w_multi_tests.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/r2w_multi_tests.log
for f in 0 1; do
  ODMOE_P2P_FUSED=$f timeout 900 $TR --master-port 2954$f bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 > gpurun_out/r2w_bench_f$f.json 2> gpurun_out/r2w_bench_f$f.err; echo "bench fused_send=$f rc=$?"
  python - $f <<'P'
import json, sys
b = json.load(open(f"gpurun_out/r2w_bench_f{sys.argv[1]}.json"))
print("fused_send", sys.argv[1], "tok/s", round(b["value"], 3), "link", round(b["host_link"]["frac"], 3), "us/expert", [round(x, 1) for x in b["roofline"]["us_per_expert_by_rank"]],
      "resident", round(b["resident"]["value"], 1), "res us/expert", round(b["roofline_resident"]["avg_us_per_expert"], 1))
P
done
