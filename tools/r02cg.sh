set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02cg_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02cg_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cg_smoke.log 2>&1; tail -2 gpurun_out/r02cg_smoke.log
timeout 600 python bench.py > gpurun_out/r02cg_bench.log 2>&1; tail -c 300 gpurun_out/r02cg_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02cg_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02cg_ncu.log 2>&1; echo ncu=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_op_hmma_src_fp16_dst_fp32_sparsity_off.sum,sm__ops_path_tensor_op_hmma_src_tf32_dst_fp32_sparsity_off.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $M --clock-control none -k regex:"conv1_fwd_ig|fc1_gram_split" -c 12 --csv --log-file gpurun_out/r02cg_metrics.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02cg_ncu2.log 2>&1; echo ncu2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02cg_ref.log 2>&1; tail -c 300 gpurun_out/r02cg_ref.log
