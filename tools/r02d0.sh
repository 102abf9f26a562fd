set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02d0_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02d0_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d0_smoke.log 2>&1; tail -2 gpurun_out/r02d0_smoke.log
timeout 600 python bench.py > gpurun_out/r02d0_bench.log 2>&1; tail -c 300 gpurun_out/r02d0_bench.log
timeout 900 python bench.py --workload resnet --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02d0_rn_bench.log 2>&1; grep '^{' gpurun_out/r02d0_rn_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('RN', d['value'], d['ms_per_step'])"
