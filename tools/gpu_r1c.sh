#!/bin/bash
# 1-GPU: full GPU tests (NF4 / BF16 shadows, swizzled activations), kernel bench, short bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "not multi" > gpurun_out/gpu_tests_c.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/gpu_tests_c.log
timeout 300 python tools/kernel_bench.py --only gemv > gpurun_out/kb_c.json 2>&1; echo "kb rc=$?"; cat gpurun_out/kb_c.json
timeout 300 python tools/kernel_bench.py --only lm > gpurun_out/kb_c_lm.json 2>&1; cat gpurun_out/kb_c_lm.json
timeout 900 python bench.py --steps 8 --warmup 3 --prefill 0 --no-cpu-baseline > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err; echo "bench rc=$?"; cat gpurun_out/bench_c.json; tail -3 gpurun_out/bench_c.err
