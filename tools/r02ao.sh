#!/bin/bash
# conv1_bwd_w A-staging remap: CNN parity + headline bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_bench_parity.py -q -p no:warnings -x > gpurun_out/r02ao_pytest.log 2>&1
tail -3 gpurun_out/r02ao_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/r02ao_bench.log 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/r02ao_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print(d["value"], d["ms_per_step"]); print({k: round(v/d["profile_pass"]["steps"],3) for k,v in list(d["kernels_ms"].items())[:8]})
PY
