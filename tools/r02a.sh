set -x
python -m pytest tests/test_gpu_multirank.py -q -p no:warnings > gpurun_out/r02a_multirank.log 2>&1; tail -3 gpurun_out/r02a_multirank.log
python bench.py > gpurun_out/r02a_bench.log 2>&1; tail -c 600 gpurun_out/r02a_bench.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_hmma_src_fp16_dst_fp32_sparsity_off.sum,sm__ops_path_tensor_op_hmma_src_tf32_dst_fp32_sparsity_off.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:"tc_kernel|weighted_sum|row_sumsq|fc1_gram|fc1_dp_hist|dz2_build|pooled_split|noise_avg" -c 160 --csv --log-file gpurun_out/r02a_metrics.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02a_ncu.log 2>&1; echo ncu_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02a_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02a_ncu2.log 2>&1; echo ncu2_rc=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02a_ref.log 2>&1; tail -c 1500 gpurun_out/r02a_ref.log
