#!/bin/bash
# N-GPU: multi tests (groups + sliced), bench groups vs sliced (phase log on stderr), sliced sweep.
N=${1:-2}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi3_n$N.log 2>&1; echo "multi tests rc=$?"; tail -5 gpurun_out/multi3_n$N.log
for PL in sliced groups; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N --steps 12 --warmup 3 --placement $PL > gpurun_out/bench3_${PL}_n$N.json 2> gpurun_out/bench3_${PL}_n$N.err; echo "bench $PL rc=$?"
  cat gpurun_out/bench3_${PL}_n$N.json; grep "bench r0" gpurun_out/bench3_${PL}_n$N.err | tail -3
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N tools/sweep.py --placement sliced --predictors shadow_int8,perfect,none --lookaheads 1,2 --refine 0,1,2 --steps 10 --out gpurun_out/sweep3_sliced_n$N.jsonl > gpurun_out/sweep3_sliced_n$N.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep3_sliced_n$N.jsonl
