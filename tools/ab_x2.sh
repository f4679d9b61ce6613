#!/bin/bash
for rep in 1 2; do
for v in "" _x2; do
  r=$(ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so timeout 120 python tools/kernel_bench.py --only gemv --iters 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print({k:round(v['us_median'],1) for k,v in d.items()})")
  l=$(ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so timeout 120 python tools/kernel_bench.py --only lm --iters 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['lm_head_argmax']['us_median'],1))")
  echo "rep=$rep lib=libodmoe$v gemv=$r lm=$l"
done
done
ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe_x2.so timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -x -q -k "not mixtral_decode" 2>&1 | tail -3
