#!/bin/bash
# Session 2, call I: ncu --set full of the prefill grouped GEMM (GEMM1 SwiGLU + GEMM2 gate) at T=512.
mkdir -p gpurun_out
timeout 300 python tools/kernel_bench.py --only grouped --iters 4 > gpurun_out/s2i_kb.json 2>&1; echo "kb rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k grouped_gemm_kernel -s 2 -c 2 -o /tmp/gg python tools/kernel_bench.py --only grouped --iters 1 > gpurun_out/s2i_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/gg.ncu-rep --page raw --csv > gpurun_out/s2i_gg_raw.csv 2>/dev/null
ncu -i /tmp/gg.ncu-rep --page source --csv --print-source sass > gpurun_out/s2i_gg_sass.csv 2>/dev/null
ls -la gpurun_out/
