#!/bin/bash
# Session 2, call H (N GPUs): prediction communicator limited to one CTA + one SM left free by the
# flat engine at N > 1; then the fused cooperative expert kernel at N > 1 (ODMOE_FUSED_NGPU=1),
# each bounded by its own timeout.
N=${1:-2}
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
B="bench.py --gpus $N --steps 8 --warmup 3 --no-cpu-baseline --prefill 0"
timeout 600 $R --master-port 29601 $B > gpurun_out/s2h_bench_n$N.json 2> gpurun_out/s2h_bench_n$N.err; echo "bench rc=$?"
ODMOE_FUSED_NGPU=1 timeout 600 $R --master-port 29602 $B > gpurun_out/s2h_bench_fused_n$N.json 2> gpurun_out/s2h_bench_fused_n$N.err; echo "bench fused rc=$?"
python - <<PY
import json
for f in ["s2h_bench_n$N", "s2h_bench_fused_n$N"]:
    try:
        d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, round(d["value"], 3), "link", round(d["host_link"]["frac"], 4), "expert_us", round(r["avg_us_per_expert"], 1),
              "w13", round(r["w13_us"], 1), "w2", round(r["w2_us"], 1), "frac", round(r["frac"], 3), "resident", round(d["resident"]["value"], 1))
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/s2h_multi_n$N.log 2>&1; echo "multi tests rc=$?"; tail -2 gpurun_out/s2h_multi_n$N.log
ODMOE_FUSED_NGPU=1 timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/s2h_multi_fused_n$N.log 2>&1; echo "multi tests fused rc=$?"; tail -2 gpurun_out/s2h_multi_fused_n$N.log
