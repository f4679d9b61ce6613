#!/bin/bash
# Round 2, 2-GPU box (b): fused expert kernel + W2-epilogue P2P send at N > 1 (defaults now), groups
# with G=1 (N_G = 2): multi tests incl. emulation equality, the default bench at N=2, Eq. 1 with two
# groups from the trace, and the token-alignment-period sweep.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -k "2" > gpurun_out/m2b_tests.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/m2b_tests.log
timeout 900 $TR --master-port 29511 bench.py --gpus 2 --steps 12 --warmup 3 > gpurun_out/m2b_bench.json 2> gpurun_out/m2b_bench.err; echo "bench n2 rc=$?"
python -c "import json; b=json.load(open('gpurun_out/m2b_bench.json')); print(b['value'], json.dumps(b['roofline'])[:300], b['host_link']['frac'], json.dumps(b.get('resident'))[:200])"
timeout 900 $TR --master-port 29512 bench.py --gpus 2 --steps 8 --warmup 2 --placement groups --group-size 1 --lookahead 2 --refine 0 --no-resident --prefill 0 --no-cpu-baseline --no-r0 --trace-steps 3 > gpurun_out/m2b_bench_groups_g1.json 2> gpurun_out/m2b_bench_groups_g1.err; echo "bench groups G=1 rc=$?"
python -c "import json; b=json.load(open('gpurun_out/m2b_bench_groups_g1.json')); print(b['value'], json.dumps(b.get('eq1')), b['host_link']['frac'])"
timeout 1500 $TR --master-port 29513 tools/sweep.py --placement groups --group-size 1 --predictors shadow_int8,perfect --lookaheads 2 --refine 0 --periods 1,2,4 --steps 8 --warmup 2 --out gpurun_out/m2b_sweep_periods.jsonl > gpurun_out/m2b_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/m2b_sweep_periods.jsonl
