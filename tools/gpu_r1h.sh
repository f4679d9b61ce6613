#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests_h.log 2>&1; echo "attn tests rc=$?"; tail -5 gpurun_out/attn_tests_h.log
BS="python bench.py --attention --steps 2 --warmup 1 --no-resident --no-cpu-baseline --prefill 0"
timeout 600 $BS > gpurun_out/bs_attn_h.log 2>&1; echo "bs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rope|attn_|gemv_rows|combine|router_kernel|flat_gemv_kernel<__nv_bfloat16, (unsigned short, 3|float, 1)" --kernel-name-base demangled -c 400 --csv --log-file gpurun_out/launches_attn_h.csv $BS > gpurun_out/ncu_attn_h.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --attention --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn3_n1.json 2> gpurun_out/bench_attn3_n1.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_attn3_n1.err
