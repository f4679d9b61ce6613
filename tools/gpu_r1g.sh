#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py -x -q > gpurun_out/attn_tests_g.log 2>&1; echo "attn tests rc=$?"; tail -5 gpurun_out/attn_tests_g.log
BS="python bench.py --attention --steps 2 --warmup 1 --no-resident --no-cpu-baseline --prefill 64"
timeout 600 $BS > gpurun_out/bs_attn.log 2>&1; echo "bs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rope|attn|flat_gemv|gemv_rows|combine|router|flat_expert" -c 600 --csv --log-file gpurun_out/launches_attn.csv $BS > gpurun_out/ncu_attn.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --attention --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/bench_attn2_n1.json 2> gpurun_out/bench_attn2_n1.err; echo "bench rc=$?"; cat gpurun_out/bench_attn2_n1.json; tail -2 gpurun_out/bench_attn2_n1.err
