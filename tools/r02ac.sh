timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_engine.py tests/test_gpu_bench_parity.py tests/test_gpu_fedsim_dropin.py tests/test_gpu_engine_edges.py tests/test_gpu_multirank.py -q -p no:warnings 2>&1 | tail -4
timeout 600 python bench.py --steps 20 --warmup 3 --e2e-steps 5 --no-cpu-baseline > gpurun_out/r02ac_bench.log 2>&1; tail -c 300 gpurun_out/r02ac_bench.log; python -c "
import json; d=json.loads(open('gpurun_out/r02ac_bench.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
