#!/bin/bash
# Round 2, call z2 (2-GPU box): NVLink keep-alive during the warm wait: per-expert trace durations and
# N = 2 tok/s with the keep-alive on / off (fused P2P send, the default).
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for k in 1 0; do
  ODMOE_LINK_KEEPALIVE=$k timeout 900 $TR --master-port 2958$k tools/p2p_probe.py --tag keep$k > gpurun_out/p2p_probe_keep$k.log 2>&1; echo "probe keep$k rc=$?"; tail -1 gpurun_out/p2p_probe_keep$k.log
done
for k in 1 0 1 0; do
  ODMOE_LINK_KEEPALIVE=$k timeout 900 $TR --master-port 29590 bench.py --gpus 2 --steps 12 --warmup 3 --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 --no-resident > gpurun_out/r2z2_bench_k$k.json 2> gpurun_out/r2z2_bench_k$k.err
  python - $k <<'P'
import json, sys
b = json.load(open(f"gpurun_out/r2z2_bench_k{sys.argv[1]}.json"))
print("keepalive", sys.argv[1], "tok/s", round(b["value"], 4), "link frac", round(b["host_link"]["frac"], 4), "us/expert", [round(x, 1) for x in b["roofline"]["us_per_expert_by_rank"]])
P
done
