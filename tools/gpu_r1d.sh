#!/bin/bash
# 1-GPU: low-bit shadow tests, kernel A/B (fp32 vs bf16 activations for low-bit weights), ncu of the
# low-bit fused kernels, shadow-precision recall at Mixtral shape (N=1, Mode A and refined).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -m gpu -x -q -k "fp8 or nf4 or lowbit or shadow or invariance" > gpurun_out/gpu_tests_d.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_d.log
timeout 300 python tools/kernel_bench.py --only gemv > gpurun_out/kb_d_f32.json 2>&1; echo "kb rc=$?"; cat gpurun_out/kb_d_f32.json
ODMOE_LOWBIT_X=bf16 timeout 300 python tools/kernel_bench.py --only gemv > gpurun_out/kb_d_bf16.json 2>&1; cat gpurun_out/kb_d_bf16.json
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"flat_expert_kernel<(signed|odmoe::nf4|odmoe::fp8)" -c 3 -o gpurun_out/prof_lowbit python tools/kernel_bench.py --only gemv --iters 2 > gpurun_out/ncu_lowbit.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_lowbit.log
for P in shadow_int8 shadow_fp8 shadow_nf4; do
  timeout 600 python tools/sweep.py --build-predictor $P --predictors $P --lookaheads 1 --refine 0,2 --steps 16 --warmup 2 --out gpurun_out/sweep_prec_$P.jsonl > gpurun_out/sweep_prec_$P.log 2>&1; echo "sweep $P rc=$?"; cat gpurun_out/sweep_prec_$P.jsonl
done
