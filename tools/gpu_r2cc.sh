#!/bin/bash
# Round 2, call cc: loader chunk size A/B at N = 1, interleaved (tok/s against the link roofline of the same run).
mkdir -p gpurun_out
i=0
for mb in 32 128 32 128 32 128 32 128; do
  i=$((i+1))
  timeout 900 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 --no-resident --chunk-mb $mb --out gpurun_out/r2cc_bench_${mb}_$i.json > gpurun_out/r2cc_bench_${mb}_$i.log 2>&1
  python - $mb $i <<'P'
import json, sys
b = json.load(open(f"gpurun_out/r2cc_bench_{sys.argv[1]}_{sys.argv[2]}.json"))
print("chunk", sys.argv[1], "MiB tok/s", round(b["value"], 4), "link frac", round(b["host_link"]["frac"], 4), "peak", round(b["host_link"]["peak"], 2),
      "reloads", b["engine"]["reloads"])
P
done
