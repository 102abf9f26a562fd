#!/bin/bash
# LM shared first-batch eval: LM / multirank GPU tests and the lm bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lm.py tests/test_gpu_multirank.py -q -p no:warnings > gpurun_out/r02ad_pytest.log 2>&1
timeout 500 python bench.py --workload lm --steps 5 --warmup 3 --e2e-steps 0 --profile-steps 2 --no-cpu-baseline > gpurun_out/r02ad_bench.log 2>&1
tail -3 gpurun_out/r02ad_pytest.log; tail -2 gpurun_out/r02ad_bench.log
