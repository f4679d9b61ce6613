#!/bin/bash
# 1-GPU refresh: GEMV variant A/B, full GPU test suite (incl. slow), default bench, ncu launch list
# of the bench + one full capture of the fused expert kernel (kernel_bench, small footprint).
mkdir -p gpurun_out
bash tools/ab_gemv.sh > gpurun_out/ab_final.log 2>&1; cat gpurun_out/ab_final.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_final.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/gpu_tests_final.log
timeout 900 python bench.py > gpurun_out/bench_final_n1.json 2> gpurun_out/bench_final_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_final_n1.json; tail -2 gpurun_out/bench_final_n1.err
BS="python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline --prefill 0"
timeout 600 $BS > gpurun_out/bs_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flat_|router_kernel|combine|embed" -c 2000 --csv --log-file gpurun_out/launches_final.csv $BS > gpurun_out/ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/kernel_bench.py --only gemv --iters 3 > gpurun_out/kb_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"flat_expert_kernel" -c 2 -o gpurun_out/prof_fused python tools/kernel_bench.py --only gemv --iters 3 > gpurun_out/ncu_fused.log 2>&1; echo "ncu full rc=$?"
