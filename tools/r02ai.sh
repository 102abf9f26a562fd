#!/bin/bash
# ResNet-18 (config D): parity tests + bench after the im2col restructure
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -s --timeout 900 > gpurun_out/r02ai_pytest.log 2>&1
tail -3 gpurun_out/r02ai_pytest.log
grep "config D client" gpurun_out/r02ai_pytest.log
timeout 900 python bench.py --workload resnet --steps 3 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02ai_bench.log 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/r02ai_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print(d["value"], d["ms_per_step"], d["profile_pass"]["ms_per_step"]); print(json.dumps(d["kernels_ms"])[:1500])
PY
