#!/bin/bash
# Round 2, call h: lean tensor-core shadow kernel (v2), cluster router, warm wait: parity, ncu launch
# list, kernel_bench, default N=1 bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q > gpurun_out/r2h_kern.log 2>&1; echo "kern rc=$?"; tail -3 gpurun_out/r2h_kern.log
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_speculation.py tests/test_gpu_emulate.py -m gpu -q > gpurun_out/r2h_eng.log 2>&1; echo "eng rc=$?"; tail -8 gpurun_out/r2h_eng.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"mma_gemv|router_cluster" -s 64 -c 30 --csv --log-file gpurun_out/r2h_ncu.csv python tools/shadow_probe.py --passes 2 > gpurun_out/r2h_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python tools/kernel_bench.py --only shadow --iters 20 > gpurun_out/r2h_kb_shadow.json 2>&1; echo "kb rc=$?"
timeout 600 python tools/kernel_bench.py --only router --iters 20 > gpurun_out/r2h_kb_router.json 2>&1; echo "kb router rc=$?"
timeout 900 python bench.py --steps 12 --warmup 3 > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
b = json.load(open("gpurun_out/r2h_bench.json"))
for key in ("value", "roofline", "roofline_shadow", "roofline_shadow_pass", "resident", "eq1", "sep_refine0"):
    print(key, json.dumps(b.get(key))[:700])
PY
