#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py -x -q -k "kv_alignment" -s > gpurun_out/kvalign_test.log 2>&1; echo "kv test rc=$?"; grep -E "passed|failed|recall" gpurun_out/kvalign_test.log | tail -3
timeout 900 python tools/sweep.py --attention --predictors shadow_int8 --lookaheads 1 --refine 0,2 --kv-align 1,0 --steps 12 --warmup 2 --out gpurun_out/sweep_kv_n1.jsonl > gpurun_out/sweep_kv_n1.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep_kv_n1.jsonl
timeout 300 python tools/kernel_bench.py --only read > gpurun_out/kb_read.json 2>&1; cat gpurun_out/kb_read.json
ODMOE_FUSED=0 timeout 300 python tools/kernel_bench.py --only gemv --iters 3 > gpurun_out/kb_nofuse.json 2>&1 && \
ODMOE_FUSED=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"flat_gemv_kernel" -c 40 --csv --log-file gpurun_out/launches_nofuse.csv python tools/kernel_bench.py --only gemv --iters 3 > gpurun_out/ncu_nofuse.log 2>&1; echo "ncu rc=$?"
