#!/bin/bash
# warp-state stall breakdown of the conv1 tcgen05 kernels (one launch each)
mkdir -p gpurun_out
timeout 900 ncu --section WarpStateStats --section SchedulerStats --section Occupancy --section MemoryWorkloadAnalysis --clock-control none -k regex:"conv1_(fwd|bwd_w)_tc_kernel" -s 20 -c 2 --csv --page details python bench.py --steps 1 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02al_ncu.csv 2> gpurun_out/r02al_ncu.err
tail -2 gpurun_out/r02al_ncu.err
wc -l gpurun_out/r02al_ncu.csv
