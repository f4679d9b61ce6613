#!/bin/bash
# Round 2, 4-GPU box: multi tests (N=4), default bench at N=4 (sliced), the paper's groups at N=4
# (G=2, N_G=2; Eq. 1 from the trace), and the alignment-period sweep on the paper's groups.
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests/test_gpu_multi.py -q -k "4" > gpurun_out/m4_tests.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/m4_tests.log
timeout 900 $TR --master-port 29521 bench.py --gpus 4 --steps 12 --warmup 3 > gpurun_out/m4_bench.json 2> gpurun_out/m4_bench.err; echo "bench n4 rc=$?"
python -c "import json; b=json.load(open('gpurun_out/m4_bench.json')); print(b['value'], b['host_link']['frac'], json.dumps(b['roofline'])[:250], json.dumps(b.get('resident'))[:150])"
timeout 900 $TR --master-port 29522 bench.py --gpus 4 --steps 8 --warmup 2 --placement groups --lookahead 2 --refine 2 --no-resident --prefill 0 --no-cpu-baseline --trace-steps 3 > gpurun_out/m4_bench_groups.json 2> gpurun_out/m4_bench_groups.err; echo "bench groups rc=$?"
python -c "import json; b=json.load(open('gpurun_out/m4_bench_groups.json')); print(b['value'], b['host_link']['frac'], json.dumps(b.get('eq1')), json.dumps(b.get('sep_refine0')))"
timeout 1800 $TR --master-port 29523 tools/sweep.py --placement groups --predictors shadow_int8,perfect --lookaheads 2 --refine 0 --periods 1,2,4 --steps 8 --warmup 2 --out gpurun_out/m4_sweep_periods.jsonl > gpurun_out/m4_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/m4_sweep_periods.jsonl
