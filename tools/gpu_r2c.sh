#!/bin/bash
# Round 2, call c: speculation tests, then the default bench (N=1) with the new legs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_speculation.py -q > gpurun_out/r2c_spec.log 2>&1; echo "spec rc=$?"; tail -25 gpurun_out/r2c_spec.log
timeout 900 python bench.py --steps 12 --warmup 3 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$?"; cat gpurun_out/r2c_bench.json; tail -5 gpurun_out/r2c_bench.err
