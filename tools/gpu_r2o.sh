#!/bin/bash
# Round 2, call o: decode router v2 (one split cluster barrier, remote mbarrier arrive to CTA 0):
# parity (router + engine tests), launch-list A/B cluster vs one-CTA, memcheck of the cluster kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -x > gpurun_out/r2o_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2o_tests.log
timeout 300 compute-sanitizer --tool memcheck python tools/kernel_bench.py --only router --iters 2 > gpurun_out/r2o_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/r2o_memcheck.log
timeout 300 compute-sanitizer --tool racecheck python tools/kernel_bench.py --only router --iters 2 > gpurun_out/r2o_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/r2o_racecheck.log
for v in 1 0; do
  ODMOE_ROUTER_CLUSTER=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"router" -c 10 --csv --log-file gpurun_out/r2o_router_list$v.csv python tools/kernel_bench.py --only router --iters 6 > gpurun_out/r2o_list$v.log 2>&1; echo "list cluster=$v rc=$?"
  grep -o '"gpu__time_duration.sum","nsecond","[0-9.,]*"' gpurun_out/r2o_router_list$v.csv | tail -6
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"router_cluster" -s 3 -c 1 -o gpurun_out/r2o_router_cluster python tools/kernel_bench.py --only router --iters 4 > gpurun_out/r2o_ncu1.log 2>&1; echo "ncu cluster rc=$?"
