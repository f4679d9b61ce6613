#!/bin/bash
# Session 2, call K (4 GPUs): configs[2] lookahead x predictor sweep with the final build, the paper's
# worker groups and the sliced placement.
N=${1:-4}
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 $R --master-port 29611 tools/sweep.py --placement groups --predictors shadow_int8,perfect,none,random --lookaheads 1,2,3,4 --refine 0,2 --steps 8 --out gpurun_out/s2k_sweep_groups_n$N.jsonl > gpurun_out/s2k_sweep_groups_n$N.log 2>&1; echo "sweep groups rc=$?"
timeout 900 $R --master-port 29612 tools/sweep.py --placement sliced --predictors shadow_int8,perfect,none,random --lookaheads 1,2 --refine 0,2 --steps 8 --out gpurun_out/s2k_sweep_sliced_n$N.jsonl > gpurun_out/s2k_sweep_sliced_n$N.log 2>&1; echo "sweep sliced rc=$?"
python - <<PY
import json
for f in ["s2k_sweep_groups_n$N", "s2k_sweep_sliced_n$N"]:
    try:
        for line in open(f"gpurun_out/{f}.jsonl"):
            d = json.loads(line)
            print(f[10:], {k: (round(v, 3) if isinstance(v, float) else v) for k, v in d.items() if k in ("predictor", "lookahead", "refine_depth", "tok_s", "h2d_GBps_aggregate", "recall_eq3", "recall_refined", "wasted_bytes_per_token")})
    except Exception as e:
        print(f, "ERR", e)
PY
