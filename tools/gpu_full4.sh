#!/bin/bash
N=${1:-4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi_tests3_n$N.log 2>&1; echo "multi tests rc=$?"; tail -3 gpurun_out/multi_tests3_n$N.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N --steps 16 --warmup 3 > gpurun_out/bench_full_n$N.json 2> gpurun_out/bench_full_n$N.err; echo "bench rc=$?"
cat gpurun_out/bench_full_n$N.json; tail -3 gpurun_out/bench_full_n$N.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus $N --steps 256 --warmup 3 --prefill 512 --no-resident > gpurun_out/bench_c5_n$N.json 2> gpurun_out/bench_c5_n$N.err; echo "c5 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_c5_n$N.json'))
print('C5 N=$N decode tok/s', d['value'], 'ttft ms', d['prefill']['ttft_ms_rank'], 'recall', d['recall_eq3'], d['recall_refined'])
"
