#!/bin/bash
mkdir -p gpurun_out
BS="python bench.py --attention --steps 2 --warmup 1 --no-cpu-baseline --prefill 0 --slots -1"
timeout 600 $BS > gpurun_out/bs_res_attn.log 2>&1; echo "bs rc=$?"; tail -2 gpurun_out/bs_res_attn.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"rope|attn_|flat_gemv|flat_expert|combine|router|embed" -c 1500 --csv --log-file gpurun_out/launches_res_attn.csv $BS > gpurun_out/ncu_res_attn.log 2>&1; echo "ncu rc=$?"
