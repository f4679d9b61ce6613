#!/bin/bash
# 1-GPU: full GPU test suite, default bench (multi-expert resident launch, stream priorities).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_e.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_e.log
timeout 900 python bench.py > gpurun_out/bench_e_n1.json 2> gpurun_out/bench_e_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_e_n1.json; grep "bench r0" gpurun_out/bench_e_n1.err | tail -2
