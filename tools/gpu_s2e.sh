#!/bin/bash
# Session 2, call E: prefill GEMM1 tile width 224 (wave quantisation) -- parity tests + A/B vs 256;
# on-demand split (non-cooperative) expert launches vs fused (launch-latency check).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefill.py -x -q -m gpu > gpurun_out/s2e_prefill_tests.log 2>&1; echo "prefill tests rc=$?"; tail -2 gpurun_out/s2e_prefill_tests.log
for bn in 224 256; do
  ODMOE_GG_BN=$bn timeout 300 python tools/kernel_bench.py --only grouped --iters 20 > gpurun_out/s2e_gg_$bn.json 2>/dev/null
  echo "gg BN=$bn: $(python -c "import json; d=json.load(open('gpurun_out/s2e_gg_$bn.json'))['grouped_ffn_T512']; print(round(d['ms_median'],3), 'ms', round(d['TFLOPs']), 'TFLOP/s', round(d['frac_hbm'],3), 'of HBM')")"
done
B="python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-resident"
timeout 900 $B --prefill 512 > gpurun_out/s2e_bench_prefill.json 2> gpurun_out/s2e_bench_prefill.err; echo "bench prefill rc=$?"
ODMOE_FUSED=0 timeout 900 $B --prefill 0 > gpurun_out/s2e_bench_split.json 2> gpurun_out/s2e_bench_split.err; echo "bench split rc=$?"
python - <<'PY'
import json
for f in ["s2e_bench_prefill", "s2e_bench_split"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, round(d["value"], 3), "expert_us", round(r["avg_us_per_expert"], 1), "w13", round(r["w13_us"], 1), "w2", round(r["w2_us"], 1),
              "prefill", {k: v for k, v in d.get("prefill", {}).items() if k != "note"})
    except Exception as e:
        print(f, "ERR", e)
PY
