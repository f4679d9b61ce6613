#!/bin/bash
# 4-GPU: all multi tests (groups, sliced incl. resident, attention), benches sliced / groups / sliced+attention.
N=${1:-4}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/multi5_n$N.log 2>&1; echo "multi tests rc=$?"; tail -5 gpurun_out/multi5_n$N.log
run_bench() {
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $3 bench.py --gpus $N --steps 16 --warmup 3 $2 > gpurun_out/bench5_$1_n$N.json 2> gpurun_out/bench5_$1_n$N.err; echo "bench $1 rc=$?"
  cat gpurun_out/bench5_$1_n$N.json; grep "bench r0" gpurun_out/bench5_$1_n$N.err | tail -2
}
run_bench sliced "--placement sliced" 29581
run_bench groups "--placement groups --prefill 0 --no-cpu-baseline" 29582
run_bench sliced_attn "--placement sliced --attention --steps 8" 29583
