set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cb_smoke.log 2>&1; tail -3 gpurun_out/r02cb_smoke.log
timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_bench_parity.py -q -p no:warnings -x > gpurun_out/r02cb_pytest.log 2>&1; tail -5 gpurun_out/r02cb_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02cb_bench.log 2>&1; tail -c 300 gpurun_out/r02cb_bench.log
