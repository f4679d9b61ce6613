#!/bin/bash
# Round 2, 2-GPU box: multi-GPU tests (incl. real == one-GPU emulation bitwise), the default bench at
# N=2 (sliced), the paper's groups with G=1 (N_G = 2: Eq. 1 with two groups, traced), and the token
# alignment period sweep (cross-token speculation) at N=2 groups.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -k "2" > gpurun_out/m2_tests.log 2>&1; echo "multi tests rc=$?"; tail -5 gpurun_out/m2_tests.log
timeout 900 $TR --master-port 29511 bench.py --gpus 2 --steps 12 --warmup 3 > gpurun_out/m2_bench.json 2> gpurun_out/m2_bench.err; echo "bench n2 rc=$?"; head -c 600 gpurun_out/m2_bench.json; echo
timeout 900 $TR --master-port 29512 bench.py --gpus 2 --steps 8 --warmup 2 --placement groups --group-size 1 --lookahead 2 --refine 0 --no-resident --prefill 0 --no-cpu-baseline --no-r0 --trace-steps 3 > gpurun_out/m2_bench_groups_g1.json 2> gpurun_out/m2_bench_groups_g1.err; echo "bench groups G=1 rc=$?"
python -c "import json; b=json.load(open('gpurun_out/m2_bench_groups_g1.json')); print(b['value'], json.dumps(b.get('eq1')))"
timeout 1200 $TR --master-port 29513 tools/sweep.py --placement groups --group-size 1 --predictors shadow_int8,perfect --lookaheads 2 --refine 0 --periods 1,2,4 --steps 8 --warmup 2 --out gpurun_out/m2_sweep_periods.jsonl > gpurun_out/m2_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/m2_sweep_periods.jsonl
