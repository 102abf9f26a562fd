#!/bin/bash
# ResNet split-K weight gradient: parity + bench
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -s --timeout 900 > gpurun_out/r02bb_pytest.log 2>&1
tail -2 gpurun_out/r02bb_pytest.log; grep "wide32\|narrow\|config D" gpurun_out/r02bb_pytest.log | head -12
timeout 900 python bench.py --workload resnet --steps 3 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02bb_bench.log 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/r02bb_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print(d["value"], d["ms_per_step"]); print({k: round(v/d["profile_pass"]["steps"],1) for k,v in list(d["kernels_ms"].items())[:14]})
PY
