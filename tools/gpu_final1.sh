#!/bin/bash
# Round-end style verification on 1 GPU: full GPU suite, smoke, default bench, launch list, ncu full of the fused expert kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/final_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err; echo "bench rc=$?"; cat gpurun_out/final_bench_n1.json; tail -2 gpurun_out/final_bench_n1.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_ref_n1.json 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/final_ref_n1.json | cut -c1-300
BS="python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline --prefill 0"
timeout 600 $BS > gpurun_out/final_bs.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flat_|router_kernel|combine|embed" -c 2000 --csv --log-file gpurun_out/final_launches.csv $BS > gpurun_out/final_ncu_list.log 2>&1; echo "ncu list rc=$?"
timeout 300 python tools/kernel_bench.py --only gemv --iters 3 > gpurun_out/final_kb.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"flat_expert_kernel" -c 1 -o gpurun_out/final_fused python tools/kernel_bench.py --only gemv --iters 3 > gpurun_out/final_ncu_full.log 2>&1; echo "ncu full rc=$?"
