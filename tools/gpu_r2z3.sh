#!/bin/bash
# Round 2, call z3 (2-GPU box): does GPU 0's polling of the receive rows slow the worker's fused send?
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for b in 2000 128; do
  ODMOE_P2P_BACKOFF_NS=$b timeout 900 $TR --master-port 29600 tools/p2p_probe.py --tag bo$b > gpurun_out/p2p_probe_bo$b.log 2>&1; echo "probe backoff $b rc=$?"; tail -1 gpurun_out/p2p_probe_bo$b.log
done
