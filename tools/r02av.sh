#!/bin/bash
# coalesced plain-store GEMM epilogue: LM + ResNet parity, both benches
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_lm.py -q -p no:warnings -x --timeout 900 -k "not bench_shape" > gpurun_out/r02av_pytest.log 2>&1
tail -2 gpurun_out/r02av_pytest.log
timeout 900 python bench.py --workload resnet --steps 3 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02av_rn_bench.log 2>&1
timeout 600 python bench.py --workload lm --steps 5 --warmup 3 --e2e-steps 0 --profile-steps 2 --no-cpu-baseline > gpurun_out/r02av_lm_bench.log 2>&1
python - <<'PY'
import json
for f in ("gpurun_out/r02av_rn_bench.log", "gpurun_out/r02av_lm_bench.log"):
    l=[x for x in open(f) if x.startswith("{")]
    d=json.loads(l[-1]); print(f, d["value"], d["ms_per_step"]); print({k: round(v/d["profile_pass"]["steps"],1) for k,v in list(d["kernels_ms"].items())[:6]})
PY
