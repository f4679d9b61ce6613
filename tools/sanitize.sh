#!/bin/bash
# compute-sanitizer memcheck (one tool per gpurun call) on the tiny decode + prefill + kernels
mkdir -p gpurun_out
cat > /tmp/san_run.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch
from paper_2512_03927_b200 import odmoe
from inputs import TINY, gen_prompt
for kw in (dict(predictor=odmoe.PRED_SHADOW_INT8, slots_per_gpu=2, refine_depth=2, lookahead=2),
           dict(predictor=odmoe.PRED_NONE, slots_per_gpu=-1)):
    eng = odmoe.Engine(TINY.L, TINY.E, TINY.k, TINY.d, TINY.F, TINY.V, dtype=odmoe.BF16, weight_seed=2512, **kw)
    tok, counts = eng.prefill([int(x) for x in gen_prompt(TINY, 3, 40)])
    t = tok
    for _ in range(4):
        t, _ = eng.decode_step(t)
    eng.close()
    print("ok", kw)
PY
timeout 900 python /tmp/san_run.py > gpurun_out/san_plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 50 python /tmp/san_run.py > gpurun_out/memcheck.log 2>&1; echo "memcheck rc=$?"
tail -8 gpurun_out/memcheck.log
