#!/bin/bash
# Round 2, call f: the INT8 shadow's expert phases in isolation (ncu launch list), tensor-core path vs
# the CUDA-core flat engine.
mkdir -p gpurun_out
for v in 1 0; do
  ODMOE_SHADOW_MMA=$v timeout 600 python tools/shadow_probe.py --passes 4 > gpurun_out/r2f_probe$v.log 2>&1; echo "probe mma=$v rc=$?"; tail -4 gpurun_out/r2f_probe$v.log
  ODMOE_SHADOW_MMA=$v timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"mma_gemv|flat_gemv_multi" -s 64 -c 24 --csv --log-file gpurun_out/r2f_ncu$v.csv python tools/shadow_probe.py --passes 2 > gpurun_out/r2f_ncu$v.log 2>&1; echo "ncu mma=$v rc=$?"
done
