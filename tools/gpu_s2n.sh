#!/bin/bash
# Session 2, call N: ncu --set full of the dominant kernels of the on-demand step by GPU time share:
# the INT8 shadow's multi-expert W13 and W2 launches (W_U8 codes), in situ.
mkdir -p gpurun_out
BS="python bench.py --steps 1 --warmup 1 --no-resident --no-cpu-baseline --prefill 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"flat_gemv_multi_kernel" -s 20 -c 2 -o /tmp/sh $BS > gpurun_out/s2n_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/sh.ncu-rep --page raw --csv > gpurun_out/s2n_raw.csv 2>/dev/null
ls -la gpurun_out
