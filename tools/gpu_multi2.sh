#!/bin/bash
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_tests2_n$N.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/multi_tests2_n$N.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29535 tools/sweep.py --predictors shadow_int8,perfect --lookaheads 1,2,3 --refine 0,1,2 --out gpurun_out/sweep2_n$N.jsonl > gpurun_out/sweep2_n$N.log 2>&1; echo "sweep rc=$?"
grep '^{' gpurun_out/sweep2_n$N.log | python -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d['predictor'], 'D', d['lookahead'], 'R', d['refine_depth'], 'tok/s %.2f' % d['tok_s'], 'recA', d['recall_eq3'], 'recB', d['recall_refined'], 'corr/tok', d['refine_corrections_per_token'], 'waste GB %.2f' % (d['wasted_bytes_per_token']/1e9))
"
tail -2 gpurun_out/sweep2_n$N.log
