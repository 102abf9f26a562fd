#!/bin/bash
# ResNet-18 (config D): parity tests + first bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -s --timeout 900 > gpurun_out/r02af_pytest.log 2>&1
tail -5 gpurun_out/r02af_pytest.log
grep "config D client" gpurun_out/r02af_pytest.log
timeout 900 python bench.py --workload resnet --steps 3 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02af_bench.log 2>&1
tail -c 3000 gpurun_out/r02af_bench.log
