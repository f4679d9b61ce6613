#!/bin/bash
# Round 2, call a: parity-hardening tests (engine, kernels), smoke.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -m "gpu and not slow" -q > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"; tail -30 gpurun_out/r2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2a_smoke.log
