#!/bin/bash
# Round 2, call s: end-of-round verification on 1 GPU with the current defaults: full GPU suite, smoke,
# default bench + reference arm, launch list of a short bench (kernel shares of the step).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2s_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2s_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2s_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2s_smoke.log
timeout 900 python bench.py > gpurun_out/r2s_bench_n1.json 2> gpurun_out/r2s_bench_n1.err; echo "bench rc=$?"; head -c 400 gpurun_out/r2s_bench_n1.json; echo
timeout 900 python bench.py --impl reference > gpurun_out/r2s_ref_n1.json 2> gpurun_out/r2s_ref_n1.err; echo "ref rc=$?"; head -c 300 gpurun_out/r2s_ref_n1.json; echo
BS="python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline --prefill 0 --no-r0 --trace-steps 0"
timeout 600 $BS > gpurun_out/r2s_bs.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"flat_|router|mma_gemv|combine|embed|wait_flag|lm_" -c 3000 --csv --log-file gpurun_out/r2s_launches.csv $BS > gpurun_out/r2s_ncu_list.log 2>&1; echo "ncu list rc=$?"
python tools/launch_summary.py gpurun_out/r2s_launches.csv > gpurun_out/r2s_launch_summary.json 2>/dev/null; head -c 1500 gpurun_out/r2s_launch_summary.json
