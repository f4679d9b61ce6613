#!/bin/bash
# Session 2, call L: grouped GEMM ring depth per tile (more weight stages for one-A-half tiles): parity + A/B.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py -x -q -m gpu > gpurun_out/s2l_prefill.log 2>&1; echo "prefill tests rc=$?"; tail -1 gpurun_out/s2l_prefill.log
for rep in 1 2; do
for v in 1 0; do
  ODMOE_GG_DYN=$v timeout 300 python tools/kernel_bench.py --only grouped --iters 20 > gpurun_out/s2l_gg_$v.json 2>/dev/null
  echo "gg dyn=$v: $(python -c "import json; d=json.load(open('gpurun_out/s2l_gg_$v.json'))['grouped_ffn_T512']; print(round(d['ms_median'],3), 'ms', round(d['TFLOPs']), 'TFLOP/s', round(d['frac_hbm'],3), 'of HBM')")"
done
done
for v in 1 0; do
ODMOE_GG_DYN=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k grouped_gemm_kernel -s 2 -c 2 python tools/kernel_bench.py --only grouped --iters 1 > gpurun_out/s2l_ncu_$v.log 2>&1; echo "ncu dyn=$v rc=$?"; grep -E "duration|bytes_read" gpurun_out/s2l_ncu_$v.log | head -4
done
