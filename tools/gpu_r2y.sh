#!/bin/bash
# Round 2, call y: final single-GPU verification after the P2P / fp32 / deferred-load changes: full GPU
# suite, smoke, default bench + reference, and one ncu --set full capture of the bf16 fused expert kernel
# (the roofline kernel; its DRAM bytes are the bench line's `traffic`).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2y_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2y_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2y_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2y_smoke.log
timeout 900 python bench.py > gpurun_out/r2y_bench_n1.json 2> gpurun_out/r2y_bench_n1.err; echo "bench rc=$?"; head -c 300 gpurun_out/r2y_bench_n1.json; echo
timeout 900 python bench.py --impl reference > gpurun_out/r2y_ref_n1.json 2> gpurun_out/r2y_ref_n1.err; echo "ref rc=$?"
timeout 300 python tools/kernel_bench.py --only bf16 --iters 3 > gpurun_out/r2y_kb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"flat_expert_kernel" -s 2 -c 1 -o gpurun_out/r2y_expert_full python tools/kernel_bench.py --only bf16 --iters 3 > gpurun_out/r2y_ncu_full.log 2>&1; echo "ncu full rc=$?"
