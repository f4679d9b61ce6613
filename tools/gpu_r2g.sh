#!/bin/bash
# Round 2, call g: one-stream multi-expert mma shadow kernel: parity (kernels + engine shadow tests),
# ncu launch list of the shadow pass, kernel_bench (packed vs flat INT8 expert), ramp experiment.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "packed or shadow" > gpurun_out/r2g_kern.log 2>&1; echo "kern rc=$?"; tail -3 gpurun_out/r2g_kern.log
timeout 900 python -m pytest tests/test_gpu_engine.py -q -k "mid_shape or tiny_decode or mixtral_shadow or multi_launch" > gpurun_out/r2g_eng.log 2>&1; echo "eng rc=$?"; tail -3 gpurun_out/r2g_eng.log
timeout 600 python tools/shadow_probe.py --passes 4 > gpurun_out/r2g_probe.log 2>&1; tail -3 gpurun_out/r2g_probe.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"mma_gemv" -s 64 -c 24 --csv --log-file gpurun_out/r2g_ncu.csv python tools/shadow_probe.py --passes 2 > gpurun_out/r2g_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python tools/kernel_bench.py --only shadow --iters 20 > gpurun_out/r2g_kb.json 2>&1; echo "kb rc=$?"; tail -c 1500 gpurun_out/r2g_kb.json
for m in idle spin busy; do timeout 600 python tools/kernel_bench.py --only gemv --iters 12 --gap-ms 6 --gap-mode $m > gpurun_out/r2g_ramp_$m.json 2>&1; echo "ramp $m rc=$?"; python -c "import json,sys; b=json.loads(open('gpurun_out/r2g_ramp_$m.json').read().strip().splitlines()[-1]); print('$m', b['expert_ffn_bf16'])"; done
