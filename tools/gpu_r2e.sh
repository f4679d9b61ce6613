#!/bin/bash
# Round 2, call e: emulate tests, tensor-core INT8 shadow (engine tests incl. the Mixtral-shape shadow
# test), shadow A/B in the bench (flat CUDA-core engine vs mma path).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulate.py -q > gpurun_out/r2e_emu.log 2>&1; echo "emu rc=$?"; tail -4 gpurun_out/r2e_emu.log
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_speculation.py -m gpu -q -x > gpurun_out/r2e_engine.log 2>&1; echo "engine rc=$?"; tail -30 gpurun_out/r2e_engine.log
for v in 1 0; do
  ODMOE_SHADOW_MMA=$v timeout 900 python bench.py --steps 8 --warmup 2 --no-resident --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 > gpurun_out/r2e_bench_mma$v.json 2> gpurun_out/r2e_bench_mma$v.err; echo "bench mma=$v rc=$?"
  python -c "import json; b=json.load(open('gpurun_out/r2e_bench_mma$v.json')); print(json.dumps(b.get('roofline_shadow')), b['value'], b['recall_eq3'], b['recall_refined'])"
done
