#!/bin/bash
# Round 2, call b: cross-token speculation tests + engine regression.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_speculation.py -q -x > gpurun_out/r2b_spec.log 2>&1; echo "spec rc=$?"; tail -30 gpurun_out/r2b_spec.log
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_attention.py tests/test_gpu_prefill.py -m "gpu and not slow" -q > gpurun_out/r2b_engine.log 2>&1; echo "engine rc=$?"; tail -15 gpurun_out/r2b_engine.log
