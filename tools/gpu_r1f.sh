#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests.log 2>&1; echo "attn tests rc=$?"; tail -30 gpurun_out/attn_tests.log
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -m "gpu and not slow" > gpurun_out/engine_tests_f.log 2>&1; echo "engine tests rc=$?"; tail -3 gpurun_out/engine_tests_f.log
timeout 900 python bench.py --attention --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn_n1.json 2> gpurun_out/bench_attn_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_attn_n1.json; tail -3 gpurun_out/bench_attn_n1.err
