timeout 600 python -m pytest tests/test_gpu_lm.py -q -p no:warnings 2>&1 | tail -2
timeout 500 python bench.py --workload lm --steps 5 --warmup 3 --e2e-steps 0 --profile-steps 2 --no-cpu-baseline > gpurun_out/r02z_lm_bench.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02z_lm_bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step']); print(list(d['kernels_ms'].items())[:6])"
