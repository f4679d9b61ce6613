#!/bin/bash
# Session 2, call M: biased-uint8 INT8 shadow experts (W_U8): shadow parity tests, bench A/B, launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_engine.py -x -q -m gpu > gpurun_out/s2m_engine.log 2>&1; echo "engine tests rc=$?"; tail -2 gpurun_out/s2m_engine.log
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --prefill 0 --no-resident"
for v in 1 0; do
  ODMOE_SHADOW_U8=$v timeout 600 $B > gpurun_out/s2m_bench_$v.json 2> gpurun_out/s2m_bench_$v.err; echo "bench u8=$v rc=$?"
done
python - <<'PY'
import json
for v in ("1", "0"):
    d = json.loads(open(f"gpurun_out/s2m_bench_{v}.json").read().strip().splitlines()[-1])
    print("u8", v, round(d["value"], 3), "shadow_us/step", round(d["engine"]["us_shadow_per_step"]), "recall", d["recall_eq3"], d["recall_refined"])
PY
BS="python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline --prefill 0"
for v in 1 0; do
  ODMOE_SHADOW_U8=$v timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flat_gemv_multi" -c 400 --csv --log-file gpurun_out/s2m_launches_$v.csv $BS > /dev/null 2>&1; echo "ncu u8=$v rc=$?"
done
python tools/launch_summary.py gpurun_out/s2m_launches_1.csv u8 | head -30
python tools/launch_summary.py gpurun_out/s2m_launches_0.csv i8 | head -30
