#!/bin/bash
# A/B of the flat-GEMV pipeline variants within ONE box (boxes differ between calls).
for rep in 1 2; do
for v in "" _w16u8 _fastall; do
  for f in 1 0; do
    r=$(ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so ODMOE_FUSED=$f timeout 120 python tools/kernel_bench.py --only gemv --iters 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print({k:round(v['us_median'],1) for k,v in d.items()})")
    l=$(ODMOE_LIB=$PWD/paper_2512_03927_b200/libodmoe$v.so timeout 120 python tools/kernel_bench.py --only lm --iters 10 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(round(d['lm_head_argmax']['us_median'],1))")
    echo "rep=$rep lib=libodmoe$v fused=$f gemv=$r lm=$l"
  done
done
done
