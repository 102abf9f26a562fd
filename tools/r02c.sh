set -x
python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02c_pytest_gpu.log 2>&1; tail -5 gpurun_out/r02c_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; tail -3 gpurun_out/r02c_smoke.log
python bench.py > gpurun_out/r02c_bench.log 2>&1; tail -c 400 gpurun_out/r02c_bench.log
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_kernels.py -x -q -p no:warnings > gpurun_out/r02c_memcheck.log 2>&1; echo memcheck_rc=$?; tail -5 gpurun_out/r02c_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 50 python -m pytest tests/test_gpu_cnn.py -x -q -p no:warnings -k "not factored" > gpurun_out/r02c_racecheck.log 2>&1; echo racecheck_rc=$?; tail -5 gpurun_out/r02c_racecheck.log
