#!/bin/bash
# source-level stall sampling of conv1_bwd_w_tc (one launch)
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"conv1_bwd_w_tc_kernel" -s 8 -c 1 -o gpurun_out/r02an_c1w python bench.py --steps 1 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02an.log 2>&1
ncu -i gpurun_out/r02an_c1w.ncu-rep --page source --csv --print-source sass > gpurun_out/r02an_src.csv 2>/dev/null
ls -la gpurun_out/r02an*
