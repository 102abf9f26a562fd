set -x
timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_bench_parity.py tests/test_gpu_engine.py -q -p no:warnings -s > gpurun_out/r02cm_pytest.log 2>&1; tail -1 gpurun_out/r02cm_pytest.log; grep "cohort 1000\|cohort 125\|theta_1\|FAIL" gpurun_out/r02cm_pytest.log | head
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02cm_bench.log 2>&1; tail -c 200 gpurun_out/r02cm_bench.log
