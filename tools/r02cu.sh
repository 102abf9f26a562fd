set -x
timeout 1200 python -m pytest tests/test_gpu_lm.py -q -p no:warnings -x > gpurun_out/r02cu_pytest.log 2>&1; tail -1 gpurun_out/r02cu_pytest.log; grep FAIL gpurun_out/r02cu_pytest.log | head -3
timeout 600 python bench.py --workload lm --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02cu_lm_bench.log 2>&1; grep '^{' gpurun_out/r02cu_lm_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('LM', d['value'], d['ms_per_step']); print({k: round(v/d['profile_pass']['steps'],2) for k,v in list(d['kernels_ms'].items())[:12]})"
