timeout 600 python -m pytest tests/test_gpu_lm.py -q -p no:warnings 2>&1 | tail -3
cat > /tmp/lmb.py <<'PY'
import sys, json
sys.argv = ["bench.py", "--workload", "lm", "--steps", "5", "--warmup", "3", "--e2e-steps", "0", "--profile-steps", "2", "--no-cpu-baseline"]
sys.path.insert(0, ".")
from paper_2404_06430_b200 import native
pass
import bench
bench.main(sys.argv[1:])
PY
timeout 500 python /tmp/lmb.py > gpurun_out/r02x_lm_bench_tc.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02x_lm_bench_tc.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step']); print(list(d['kernels_ms'].items())[:6])"
