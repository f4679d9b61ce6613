#!/bin/bash
# Round 2, call n: decode router (m = 1) kernels: new parity tests, ncu full of the cluster kernel,
# launch-list A/B cluster vs one-CTA.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -k "router" > gpurun_out/r2n_router_tests.log 2>&1; echo "router tests rc=$?"; tail -3 gpurun_out/r2n_router_tests.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"router" -s 3 -c 1 -o gpurun_out/r2n_router_cluster python tools/kernel_bench.py --only router --iters 4 > gpurun_out/r2n_ncu1.log 2>&1; echo "ncu cluster rc=$?"
for v in 1 0; do
  ODMOE_ROUTER_CLUSTER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"router" -c 10 --csv --log-file gpurun_out/r2n_router_list$v.csv python tools/kernel_bench.py --only router --iters 6 > gpurun_out/r2n_list$v.log 2>&1; echo "list cluster=$v rc=$?"
  grep -o '"gpu__time_duration.sum","nsecond","[0-9.,]*"' gpurun_out/r2n_router_list$v.csv | tail -6
done
ls -la gpurun_out | grep r2n
