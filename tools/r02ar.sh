#!/bin/bash
# full GPU suite, smoke, default bench + launch list, and compute-sanitizer over the ResNet kernels
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02ar_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02ar_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ar_smoke.log 2>&1; tail -2 gpurun_out/r02ar_smoke.log
timeout 600 python bench.py > gpurun_out/r02ar_bench.log 2>&1; tail -c 400 gpurun_out/r02ar_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02ar_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02ar_ncu.log 2>&1; echo ncu=$?
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -x -k "narrow or deterministic or (wide32 and tcgen05 and B4) or shared" > gpurun_out/r02ar_memcheck_resnet.log 2>&1; echo memcheck=$?; tail -2 gpurun_out/r02ar_memcheck_resnet.log
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report analysis --print-limit 20 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -x -k "(narrow and tcgen05 and 1-4-0.05) or deterministic" > gpurun_out/r02ar_racecheck_resnet.log 2>&1; echo racecheck=$?; tail -2 gpurun_out/r02ar_racecheck_resnet.log
