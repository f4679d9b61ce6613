#!/bin/bash
# Round 2, call d: emulate_world parity tests + engine regression + smoke.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_emulate.py -q > gpurun_out/r2d_emu.log 2>&1; echo "emu rc=$?"; tail -40 gpurun_out/r2d_emu.log
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_speculation.py -m "gpu and not slow" -q > gpurun_out/r2d_engine.log 2>&1; echo "engine rc=$?"; tail -5 gpurun_out/r2d_engine.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/r2d_smoke.log
