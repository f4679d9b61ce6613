#!/bin/bash
# Round 2, call k: A/B of the tensor-core shadow GEMV variants (L2 bulk prefetch distance, warps):
# ncu launch list of the W13 / W2 phases in a shadow pass, per variant.
mkdir -p gpurun_out
for v in base pf1 pf2 w12u8; do
  if [ $v = base ]; then lib=paper_2512_03927_b200/libodmoe.so; else lib=paper_2512_03927_b200/libodmoe_mg_$v.so; fi
  ODMOE_LIB=$lib timeout 900 ncu --metrics gpu__time_duration.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"mma_gemv" -s 8 -c 16 --csv --log-file gpurun_out/r2k_ncu_$v.csv python tools/shadow_probe.py --passes 1 > gpurun_out/r2k_$v.log 2>&1; echo "$v rc=$?"
  python - "$v" <<'PY'
import csv, collections, sys
v = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r2k_ncu_{v}.csv")))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict); names = {}
for r in data:
    if len(r) > vi:
        per[r[idi]][r[mi]] = float(r[vi].replace(",", "")); names[r[idi]] = r[ki][:26]
agg = collections.defaultdict(list)
for i, m in per.items(): agg[names[i]].append(m["gpu__time_duration.sum"])
print(v, {k: round(sum(x) / len(x) / 1e3, 2) for k, x in agg.items()})
PY
done
