#!/bin/bash
# Session 2, call G: where the on-demand expert launch's extra ~15 us come from -- the same kernel
# after an idle GPU (--gap-ms), after an L2 full of dirty lines (--dirty, like right after an H2D
# load), both, and the default back-to-back measurement.
mkdir -p gpurun_out
for a in "" "--gap-ms 6" "--dirty" "--dirty --gap-ms 6"; do
  n=$(echo "$a" | tr -d ' -')
  timeout 300 python tools/kernel_bench.py --only gemv --iters 12 $a > gpurun_out/s2g_kb_$n.json 2>/dev/null
  echo "kb [$a]: $(python -c "import json; d=json.load(open('gpurun_out/s2g_kb_$n.json')); print({k:round(v['us_median'],1) for k,v in d.items()})" 2>&1 | tail -1)"
done
timeout 1200 python -m pytest tests/test_gpu_engine.py -x -q -m gpu -k "mixtral_shadow" > gpurun_out/s2g_mixtral_shadow.log 2>&1; echo "mixtral shadow test rc=$?"; tail -3 gpurun_out/s2g_mixtral_shadow.log
