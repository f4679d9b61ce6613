#!/bin/bash
# Round 2, call m: router ncu (full), cross-token speculation sweep at N=1, reference arm check.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"router_cluster" -s 40 -c 1 -o gpurun_out/r2m_router python tools/shadow_probe.py --passes 1 > gpurun_out/r2m_ncu_router.log 2>&1; echo "ncu router rc=$?"
timeout 1500 python tools/sweep.py --predictors shadow_int8,perfect --lookaheads 1,2 --refine 0 --periods 1,2,4 --slots 4 --steps 8 --warmup 2 --out gpurun_out/r2m_sweep_periods_n1.jsonl > gpurun_out/r2m_sweep.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/r2m_sweep_periods_n1.jsonl
timeout 600 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/r2m_ref.json 2> gpurun_out/r2m_ref.err; echo "ref rc=$?"; cat gpurun_out/r2m_ref.json
for fz in 1 0; do
  ODMOE_FUSED=$fz timeout 900 python bench.py --steps 10 --warmup 3 --no-resident --prefill 0 --no-cpu-baseline --no-r0 --trace-steps 0 > gpurun_out/r2m_bench_fused$fz.json 2> gpurun_out/r2m_bench_fused$fz.err; echo "bench N=1 fused=$fz rc=$?"
  python -c "import json; b=json.load(open('gpurun_out/r2m_bench_fused$fz.json')); r=b['roofline']; print('fused=$fz', round(b['value'],3), round(r['avg_us_per_expert'],1), round(r['w13_us'],1), round(r['w2_us'],1), round(r['frac'],3))"
done
