#!/bin/bash
# Round 2, 2-GPU box (c): A/B of the cooperative fused expert kernel at N > 1 and of the W2-epilogue
# P2P send (bench N=2, sliced), and the multi tests with the split launches (send in the flat W2).
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
echo "split multi tests: done in m2c run 1"
for fz in 1 0; do for ps in 1; do
  ODMOE_FUSED_NGPU=$fz ODMOE_P2P_FUSED=$ps timeout 900 $TR --master-port 295$fz$ps bench.py --gpus 2 --steps 10 --warmup 3 --no-resident --prefill 0 --no-cpu-baseline --no-r0 --trace-steps 0 > gpurun_out/m2c_bench_f${fz}_s${ps}.json 2> gpurun_out/m2c_bench_f${fz}_s${ps}.err; echo "bench fused=$fz send=$ps rc=$?"
  python -c "import json; b=json.load(open('gpurun_out/m2c_bench_f${fz}_s${ps}.json')); r=b['roofline']; print('fused=$fz send=$ps', round(b['value'],3), round(b['host_link']['frac'],4), round(r['avg_us_per_expert'],1), round(r['w13_us'],1), round(r['w2_us'],1), round(r['frac'],3))"
done; done
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -k "emulation and 2" > gpurun_out/m2c_tests.log 2>&1; echo "multi tests rc=$?"; tail -2 gpurun_out/m2c_tests.log
