#!/bin/bash
# 4-GPU: multi tests (groups + sliced, P2P combine), bench sliced (P2P / NCCL A/B) and groups, sliced sweep.
N=${1:-4}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi4_n$N.log 2>&1; echo "multi tests rc=$?"; tail -5 gpurun_out/multi4_n$N.log
run_bench() {  # name, extra args, env
  timeout 900 env $3 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $4 bench.py --gpus $N --steps 16 --warmup 3 $2 > gpurun_out/bench4_$1_n$N.json 2> gpurun_out/bench4_$1_n$N.err; echo "bench $1 rc=$?"
  cat gpurun_out/bench4_$1_n$N.json; grep "bench r0" gpurun_out/bench4_$1_n$N.err | tail -2
}
run_bench sliced "--placement sliced" "ODMOE_P2P=1" 29571
run_bench sliced_nccl "--placement sliced --no-cpu-baseline --prefill 0" "ODMOE_P2P=0" 29572
run_bench groups "--placement groups --prefill 0" "ODMOE_P2P=1" 29573
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29574 tools/sweep.py --placement sliced --predictors shadow_int8,perfect,none,random --lookaheads 1 --refine 0,1,2 --steps 10 --out gpurun_out/sweep4_sliced_n$N.jsonl > gpurun_out/sweep4_sliced_n$N.log 2>&1; echo "sweep rc=$?"; cat gpurun_out/sweep4_sliced_n$N.jsonl
