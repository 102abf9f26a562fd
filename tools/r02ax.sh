#!/bin/bash
# tensor-pipe evidence for the grouped tcgen05 GEMM in the LM and ResNet benches
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__ops_path_tensor_src_tf32_dst_fp32.sum,smsp__sass_inst_executed_op_utcmma.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:"gemm_tc_kernel" -s 300 -c 60 --csv python bench.py --workload lm --steps 1 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02ax_lm_ncu.csv 2> gpurun_out/r02ax_lm_ncu.err
timeout 1500 ncu --metrics $M --clock-control none -k regex:"gemm_tc_kernel" -s 600 -c 60 --csv python bench.py --workload resnet --steps 1 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02ax_rn_ncu.csv 2> gpurun_out/r02ax_rn_ncu.err
wc -l gpurun_out/r02ax_*.csv
