#!/bin/bash
# Round 2, call z (2-GPU box): per-expert kernel durations from the trace, fused P2P send off / on.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for f in 0 1; do
  ODMOE_P2P_FUSED=$f timeout 900 $TR --master-port 2957$f tools/p2p_probe.py --tag f$f > gpurun_out/p2p_probe_f$f.log 2>&1; echo "probe f$f rc=$?"; tail -1 gpurun_out/p2p_probe_f$f.log
done
