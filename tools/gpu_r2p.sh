#!/bin/bash
# Round 2, call p: fewer-slots-than-k deferral + expert_layer_period (engine tests), then the FP32
# (paper's precision) bench leg at N = 1 with 1 slot under the 1 GB budget.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py -q -x > gpurun_out/r2p_tests.log 2>&1; echo "engine tests rc=$?"; tail -3 gpurun_out/r2p_tests.log
timeout 1200 python bench.py --dtype fp32 --steps 8 --warmup 3 --out gpurun_out/r2p_bench_fp32.json > gpurun_out/r2p_bench_fp32.log 2>&1; echo "bench fp32 rc=$?"
tail -c 3000 gpurun_out/r2p_bench_fp32.log
