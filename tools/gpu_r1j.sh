#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "not multi" > gpurun_out/gpu_tests_j.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_j.log
timeout 900 python bench.py --attention --steps 8 --warmup 3 --no-cpu-baseline --prefill 0 > gpurun_out/bench_attn4_n1.json 2> gpurun_out/bench_attn4_n1.err; echo "bench attn rc=$?"; tail -1 gpurun_out/bench_attn4_n1.err
timeout 900 python bench.py > gpurun_out/bench_j_n1.json 2> gpurun_out/bench_j_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_j_n1.json; tail -1 gpurun_out/bench_j_n1.err
