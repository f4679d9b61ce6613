#!/bin/bash
# Session 2, call A: shadow multi-expert launches + branch-free consume. GPU engine tests, low-bit
# kernel A/B (fast vs slow consume), bench A/B (multi vs per-expert shadow launches), on-demand
# expert timing without the shadow (contention check), ncu of the in-situ INT8 multi kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/s2a_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s2a_tests.log
for v in "" _slow; do
  ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so timeout 300 python tools/kernel_bench.py --only gemv --iters 10 > gpurun_out/s2a_kb$v.json 2>/dev/null
  echo "kb$v: $(python -c "import json; d=json.load(open('gpurun_out/s2a_kb$v.json')); print({k:round(v['us_median'],1) for k,v in d.items()})")"
done
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --prefill 0 --no-resident"
timeout 600 $B > gpurun_out/s2a_bench.json 2> gpurun_out/s2a_bench.err; echo "bench rc=$?"
ODMOE_MULTI=0 timeout 600 $B > gpurun_out/s2a_bench_m0.json 2> gpurun_out/s2a_bench_m0.err; echo "bench m0 rc=$?"
timeout 600 $B --predictor none --refine 0 > gpurun_out/s2a_bench_none.json 2> gpurun_out/s2a_bench_none.err; echo "bench none rc=$?"
timeout 600 $B --refine 0 > gpurun_out/s2a_bench_r0.json 2> gpurun_out/s2a_bench_r0.err; echo "bench r0 rc=$?"
python - <<'PY'
import json
for f in ["s2a_bench", "s2a_bench_m0", "s2a_bench_none", "s2a_bench_r0"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"], 3), "expert_us", round(d["roofline"]["avg_us_per_expert"], 1), "shadow_us/step",
              round(d["engine"]["us_shadow_per_step"]), "recall", d["recall_eq3"], d["recall_refined"], "launches", d["gpu_launches"])
    except Exception as e:
        print(f, "ERR", e)
PY
BS="python bench.py --steps 1 --warmup 1 --no-resident --no-cpu-baseline --prefill 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"flat_gemv_multi_kernel" -s 4 -c 2 -o gpurun_out/s2a_multi $BS > gpurun_out/s2a_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/s2a_ncu.log
