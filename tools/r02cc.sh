set -x
timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_bench_parity.py -q -p no:warnings -s > gpurun_out/r02cc_pytest.log 2>&1; tail -3 gpurun_out/r02cc_pytest.log; grep "cohort 1000\|cohort 125\|theta_1" gpurun_out/r02cc_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02cc_bench.log 2>&1; tail -c 200 gpurun_out/r02cc_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv1_fwd_ig -s 12 -c 1 -o gpurun_out/r02cc_c1ig python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 0 > gpurun_out/r02cc_ncu.log 2>&1; echo ncu=$?
