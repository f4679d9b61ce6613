#!/bin/bash
# Round 2, call j: persistent grouped GEMM (prefill) parity + timing; full 1-GPU regression.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_attention.py -q > gpurun_out/r2j_prefill.log 2>&1; echo "prefill rc=$?"; tail -3 gpurun_out/r2j_prefill.log
timeout 600 python tools/kernel_bench.py --only grouped --iters 20 > gpurun_out/r2j_kb_grouped.json 2>&1; echo "kb rc=$?"; cat gpurun_out/r2j_kb_grouped.json | tail -12
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"grouped_gemm" -c 6 --csv --log-file gpurun_out/r2j_ncu_gg.csv python tools/kernel_bench.py --only grouped --iters 2 > gpurun_out/r2j_ncu_gg.log 2>&1; echo "ncu rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2j_all.log 2>&1; echo "all gpu rc=$?"; tail -5 gpurun_out/r2j_all.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"mma_gemv" -s 6 -c 2 -o gpurun_out/r2i_mma python tools/shadow_probe.py --passes 1 > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/ | grep r2i
