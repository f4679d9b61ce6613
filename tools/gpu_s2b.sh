#!/bin/bash
# Session 2, call B: flat-GEMV warp/unroll variants for the low-bit shadow kernels + ncu of the INT8
# shadow expert kernel (stall breakdown, source lines). Reports exported to CSV on the box.
mkdir -p gpurun_out
for v in "" _slow _w24u4 _w20u6 _w32u4 _w24u6; do
  ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so timeout 300 python tools/kernel_bench.py --only gemv --iters 10 > gpurun_out/s2b_kb$v.json 2>/dev/null
  echo "kb$v: $(python -c "import json; d=json.load(open('gpurun_out/s2b_kb$v.json')); print({k:round(v['us_median'],1) for k,v in d.items()})" 2>&1 | tail -1)"
done
for v in "" _w20u6; do
  timeout 300 python tools/kernel_bench.py --only shadow --iters 2 > /dev/null 2>&1 && \
  ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"flat_expert_kernel<signed char, float" -c 1 -o /tmp/i8$v python tools/kernel_bench.py --only shadow --iters 2 > gpurun_out/s2b_ncu$v.log 2>&1; echo "ncu$v rc=$?"
  ncu -i /tmp/i8$v.ncu-rep --page raw --csv > gpurun_out/s2b_i8$v_raw.csv 2>/dev/null
  ncu -i /tmp/i8$v.ncu-rep --page source --csv --print-source sass > gpurun_out/s2b_i8${v}_sass.csv 2>/dev/null
  ncu -i /tmp/i8$v.ncu-rep --page raw --csv > gpurun_out/s2b_i8${v}_raw.csv 2>/dev/null
  ls -la gpurun_out/s2b_i8${v}_*
done
du -sh gpurun_out
