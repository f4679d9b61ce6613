#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_prefill.py -x -q -m "gpu and not slow" > gpurun_out/tests_m.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tests_m.log
timeout 900 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --prefill 0 > gpurun_out/bench_m_n1.json 2> gpurun_out/bench_m_n1.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_m_n1.err
ODMOE_GRAPH=0 timeout 900 python bench.py --steps 16 --warmup 3 --no-cpu-baseline --prefill 0 > gpurun_out/bench_m0_n1.json 2> gpurun_out/bench_m0_n1.err; echo "bench nograph rc=$?"
python -c "
import json
for f in ['gpurun_out/bench_m_n1.json','gpurun_out/bench_m0_n1.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['value'], d['resident'])"
