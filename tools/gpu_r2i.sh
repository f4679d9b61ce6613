#!/bin/bash
# Round 2, call i: ncu --set full of the tensor-core shadow phases (W13 and W2, 2 experts) in a shadow pass.
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"mma_gemv" -s 6 -c 2 -o gpurun_out/r2i_mma python tools/shadow_probe.py --passes 1 > gpurun_out/r2i_ncu.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/ | grep r2i
