#!/bin/bash
# Round 2, call q: bf16 expert phases on the tensor cores (flat engine kMMA branch): parity, A/B vs the
# FFMA2 stream (kernel bench + ncu launch lists), N = 1 bench.
mkdir -p gpurun_out
for v in 1 0; do
  ODMOE_MAIN_MMA=$v timeout 300 python tools/kernel_bench.py --only bf16 --iters 30 > gpurun_out/r2q_kb_bf16_$v.json 2> gpurun_out/r2q_kb_bf16_$v.err; echo "kb mma=$v rc=$?"; cat gpurun_out/r2q_kb_bf16_$v.json | head -c 600; echo
done
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py tests/test_gpu_emulate.py -q -x > gpurun_out/r2q_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r2q_tests.log
for v in 1 0; do
  ODMOE_MAIN_MMA=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flat_expert" -c 12 --csv --log-file gpurun_out/r2q_list$v.csv python tools/kernel_bench.py --only bf16 --iters 6 > gpurun_out/r2q_list$v.log 2>&1; echo "list mma=$v rc=$?"
  grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' gpurun_out/r2q_list$v.csv | tail -6
done
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --prefill 0 --out gpurun_out/r2q_bench_n1.json > gpurun_out/r2q_bench_n1.log 2>&1; echo "bench rc=$?"
python - <<'P'
import json
d=json.load(open("gpurun_out/r2q_bench_n1.json"))
print("value", d["value"], "frac", d["roofline"]["frac"], "us/expert", d["roofline"]["avg_us_per_expert"])
print("resident", d.get("resident",{}).get("value"), "res frac", d.get("roofline_resident",{}).get("frac"), d.get("roofline_resident",{}).get("avg_us_per_expert"))
P
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"flat_expert" -s 3 -c 1 -o gpurun_out/r2q_expert_mma python tools/kernel_bench.py --only bf16 --iters 4 > gpurun_out/r2q_ncu_full.log 2>&1; echo "ncu full rc=$?"
