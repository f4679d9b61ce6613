#!/bin/bash
# Round 2, call r: L2 bulk prefetch of the W2 phase's next groups before the W13 -> W2 grid barrier
# (ODMOE_BARRIER_PF groups per warp): kernel bench + ncu launch list + N = 1 bench (on-demand and resident).
mkdir -p gpurun_out
for v in 0 8 16 32; do
  ODMOE_BARRIER_PF=$v timeout 300 python tools/kernel_bench.py --only bf16 --iters 40 > gpurun_out/r2r_kb_$v.json 2>/dev/null
  ODMOE_BARRIER_PF=$v timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"flat_expert" -c 10 --csv --log-file gpurun_out/r2r_list$v.csv python tools/kernel_bench.py --only bf16 --iters 6 > /dev/null 2>&1
  python - "$v" <<'P'
import json, sys, csv
v = sys.argv[1]
d = json.load(open(f"gpurun_out/r2r_kb_{v}.json"))["expert_ffn_bf16"]
t, b = [], []
for r in csv.reader(open(f"gpurun_out/r2r_list{v}.csv")):
    if len(r) > 10 and r[-3] == "gpu__time_duration.sum": t.append(float(r[-1].replace(",", "")))
    if len(r) > 10 and r[-3] == "dram__bytes_read.sum": b.append(float(r[-1].replace(",", "")))
print(f"pf={v}: events median {d['us_median']:.1f} us best {d['us_best']:.1f}; ncu list {sum(t)/max(1,len(t))/1e3:.1f} us dram {sum(b)/max(1,len(b)):.1f}")
P
done
for v in 0 16; do
  ODMOE_BARRIER_PF=$v timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 --out gpurun_out/r2r_bench_$v.json > gpurun_out/r2r_bench_$v.log 2>&1; echo "bench pf=$v rc=$?"
  python - "$v" <<'P'
import json, sys
d = json.load(open(f"gpurun_out/r2r_bench_{sys.argv[1]}.json"))
print("value", round(d["value"], 3), "frac", round(d["roofline"]["frac"], 3), "us/expert", round(d["roofline"]["avg_us_per_expert"], 1),
      "resident", round(d["resident"]["value"], 1), "res frac", round(d["roofline_resident"]["frac"], 3))
P
done
