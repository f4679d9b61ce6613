#!/bin/bash
# bench.py stdout must be the JSON line alone under torchrun (NCCL's banner goes to stderr).
mkdir -p gpurun_out
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 bench.py --gpus 2 --steps 4 --warmup 3 > gpurun_out/stdout_n2.txt 2> gpurun_out/stdout_n2.err; echo "bench rc=$?"
wc -l gpurun_out/stdout_n2.txt; python -c "import json; [json.loads(l) for l in open('gpurun_out/stdout_n2.txt')]; print('stdout is JSON only')"
