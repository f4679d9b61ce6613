#!/bin/bash
# Re-entry verification on a fresh box: GPU test suite, smoke(), default bench (N=1).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_verify.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_verify.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_verify.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_verify.log
timeout 600 python bench.py > gpurun_out/bench_verify_n1.json 2> gpurun_out/bench_verify_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_verify_n1.json; tail -2 gpurun_out/bench_verify_n1.err
