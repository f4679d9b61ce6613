#!/bin/bash
# Round-1 measurement call: Mixtral-scale parity, bench, ncu launch list + full capture of the GEMVs.
mkdir -p gpurun_out
BSMALL="python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline"
timeout 900 python -m pytest tests -m slow -x -q > gpurun_out/slow.log 2>&1; echo "slow rc=$?"
timeout 900 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?"
timeout 600 $BSMALL > gpurun_out/b_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"w13|w2_gemv|router|lm_head|embed|combine" -c 1200 --csv --log-file gpurun_out/launches.csv $BSMALL > gpurun_out/ncu1.log 2>&1; echo "ncu-list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"w13_swiglu_kernel<__nv_bfloat16|w2_gemv_kernel<__nv_bfloat16" -s 20 -c 4 -o gpurun_out/prof_gemv $BSMALL > gpurun_out/ncu2.log 2>&1; echo "ncu-full rc=$?"
tail -3 gpurun_out/slow.log; cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.err
