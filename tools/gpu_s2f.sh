#!/bin/bash
# Session 2, call F: prefill grouped GEMM with two CTAs per SM (128-wide tiles, 2-stage ring) vs
# one (256-wide, 3 stages): parity tests under both, A/B timing; mid-shape engine tests.
mkdir -p gpurun_out
for v in 0 1; do
  ODMOE_GG_2CTA=$v timeout 900 python -m pytest tests/test_gpu_prefill.py -x -q -m gpu > gpurun_out/s2f_prefill_$v.log 2>&1; echo "prefill tests 2cta=$v rc=$?"; tail -1 gpurun_out/s2f_prefill_$v.log
  ODMOE_GG_2CTA=$v timeout 300 python tools/kernel_bench.py --only grouped --iters 20 > gpurun_out/s2f_gg_$v.json 2>/dev/null
  echo "gg 2cta=$v: $(python -c "import json; d=json.load(open('gpurun_out/s2f_gg_$v.json'))['grouped_ffn_T512']; print(round(d['ms_median'],3), 'ms', round(d['TFLOPs']), 'TFLOP/s', round(d['frac_hbm'],3), 'of HBM')")"
done
timeout 900 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "mid_shape or multi_launch" > gpurun_out/s2f_mid.log 2>&1; echo "mid tests rc=$?"; tail -2 gpurun_out/s2f_mid.log
