#!/bin/bash
# Round 2, call l: fused (cooperative) tensor-core shadow layer: parity, ncu launch list, bench N=1.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_engine.py tests/test_gpu_speculation.py tests/test_gpu_emulate.py -m gpu -q > gpurun_out/r2l_eng.log 2>&1; echo "eng rc=$?"; tail -4 gpurun_out/r2l_eng.log
timeout 600 python tools/shadow_probe.py --passes 4 > gpurun_out/r2l_probe.log 2>&1; tail -3 gpurun_out/r2l_probe.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"mma_layer|router_cluster" -s 16 -c 20 --csv --log-file gpurun_out/r2l_ncu.csv python tools/shadow_probe.py --passes 2 > gpurun_out/r2l_ncu.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --steps 12 --warmup 3 > gpurun_out/r2l_bench.json 2> gpurun_out/r2l_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
b = json.load(open("gpurun_out/r2l_bench.json"))
for key in ("value", "roofline", "roofline_shadow", "roofline_shadow_pass", "resident", "eq1", "recall_eq3", "recall_refined"):
    print(key, json.dumps(b.get(key))[:500])
PY
