#!/bin/bash
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pattern_bench tools/pattern_bench.cu && timeout 300 /tmp/pattern_bench > gpurun_out/pattern_bench.json 2>&1; echo "rc=$?"; cat gpurun_out/pattern_bench.json
