set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02ct_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02ct_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ct_smoke.log 2>&1; tail -2 gpurun_out/r02ct_smoke.log
timeout 600 python bench.py > gpurun_out/r02ct_bench.log 2>&1; tail -c 300 gpurun_out/r02ct_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02ct_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02ct_ncu.log 2>&1; echo ncu=$?
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $M --clock-control none -k regex:"conv1_fwd_ig|fc1_tc" -c 20 --csv --log-file gpurun_out/r02ct_metrics.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02ct_ncu2.log 2>&1; echo ncu2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02ct_ref.log 2>&1; tail -c 300 gpurun_out/r02ct_ref.log
