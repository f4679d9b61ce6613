#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_engine.py -x -q -m "gpu and not slow" > gpurun_out/tests_l.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_l.log
timeout 900 python bench.py --attention --steps 8 --warmup 3 --no-cpu-baseline --prefill 0 > gpurun_out/bench_attn5_n1.json 2> gpurun_out/bench_attn5_n1.err; echo "bench attn rc=$?"; tail -1 gpurun_out/bench_attn5_n1.err
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --prefill 0 > gpurun_out/bench_l_n1.json 2> gpurun_out/bench_l_n1.err; echo "bench rc=$?"; tail -1 gpurun_out/bench_l_n1.err
BS="python bench.py --attention --steps 2 --warmup 1 --no-cpu-baseline --prefill 0 --slots -1"
timeout 600 $BS > gpurun_out/bs_res_attn2.log 2>&1; echo "bs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"rope|attn_|flat_gemv|flat_expert|combine|router" -c 600 --csv --log-file gpurun_out/launches_res_attn2.csv $BS > gpurun_out/ncu_res_attn2.log 2>&1; echo "ncu rc=$?"
