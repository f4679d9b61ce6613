#!/bin/bash
# Round 2, call aa: decode router with st.async + mbarrier exchanges (no cluster barrier on the path):
# parity (kernels + engine), launch-list A/B against the one-CTA router on the same box.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x > gpurun_out/r2aa_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2aa_tests.log
for v in 1 0; do
  ODMOE_ROUTER_CLUSTER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"router" -c 10 --csv --log-file gpurun_out/r2aa_router_list$v.csv python tools/kernel_bench.py --only router --iters 6 > gpurun_out/r2aa_list$v.log 2>&1; echo "list cluster=$v rc=$?"
  python tools/launch_summary.py gpurun_out/r2aa_router_list$v.csv | grep -E '"kernel"|avg_us'
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"router_cluster" -s 3 -c 1 -o gpurun_out/r2aa_router_cluster python tools/kernel_bench.py --only router --iters 4 > gpurun_out/r2aa_ncu1.log 2>&1; echo "ncu rc=$?"
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0 --out gpurun_out/r2aa_bench.json > gpurun_out/r2aa_bench.log 2>&1; echo "bench rc=$?"
python -c "import json; b=json.load(open('gpurun_out/r2aa_bench.json')); print('tok/s', b['value'], 'router us', b['engine']['us_router'], 'resident', b['resident']['value'])"
