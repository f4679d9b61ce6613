#!/bin/bash
# Session 2, call C: 24-warp x 4-granule flat GEMV as the default; warp/unroll variants; bench
# (on-demand + resident) default vs the old 16 x 8; ncu of the INT8 shadow expert; GPU tests.
mkdir -p gpurun_out
L=$PWD/paper_2512_03927_b200
for v in "" _fastall _w16u8 _w28u4 _w24u5 _w20u4; do
  ODMOE_LIB=$L/libodmoe$v.so timeout 300 python tools/kernel_bench.py --only gemv --iters 10 > gpurun_out/s2c_kb$v.json 2>/dev/null
  ODMOE_LIB=$L/libodmoe$v.so timeout 300 python tools/kernel_bench.py --only lm --iters 10 > gpurun_out/s2c_lm$v.json 2>/dev/null
  echo "kb$v: $(python -c "import json; d=json.load(open('gpurun_out/s2c_kb$v.json')); d.update(json.load(open('gpurun_out/s2c_lm$v.json'))); print({k:round(v['us_median'],1) for k,v in d.items()})" 2>&1 | tail -1)"
done
timeout 300 ncu --set full --clock-control none --import-source on -k flat_expert_kernel -c 1 -o /tmp/i8 python tools/kernel_bench.py --only shadow --iters 1 > gpurun_out/s2c_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/i8.ncu-rep --page raw --csv > gpurun_out/s2c_i8_raw.csv 2>/dev/null
ncu -i /tmp/i8.ncu-rep --page source --csv --print-source sass > gpurun_out/s2c_i8_sass.csv 2>/dev/null
ls -la gpurun_out/s2c_i8_*
B="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --prefill 0"
for v in "" _w16u8; do
  ODMOE_LIB=$L/libodmoe$v.so timeout 900 $B > gpurun_out/s2c_bench$v.json 2> gpurun_out/s2c_bench$v.err; echo "bench$v rc=$?"
done
python - <<'PY'
import json
for f in ["s2c_bench", "s2c_bench_w16u8"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        print(f, round(d["value"], 3), "expert_us", round(d["roofline"]["avg_us_per_expert"], 1), "shadow_us/step",
              round(d["engine"]["us_shadow_per_step"]), "recall", d["recall_eq3"], d["recall_refined"],
              "resident", round(d["resident"]["value"], 1), round(d["resident"]["expert_gemv_us"], 1))
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/s2c_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s2c_tests.log
du -sh gpurun_out
