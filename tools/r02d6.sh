bsum() { python - "$1" <<'PY'
import json,sys
d=[json.loads(x) for x in open(sys.argv[1]) if x.startswith("{")][-1]
print(d["value"], d["ms_per_step"]); print({k: round(v/d["profile_pass"]["steps"],3) for k,v in list(d["kernels_ms"].items())[:6]})
PY
}
timeout 900 python -m pytest tests/test_gpu_cnn.py tests/test_gpu_bench_parity.py tests/test_gpu_multirank.py -q -p no:warnings -s > gpurun_out/r02d6_pytest.log 2>&1; tail -1 gpurun_out/r02d6_pytest.log; grep "cohort 1000\|cohort 125\|FAIL" gpurun_out/r02d6_pytest.log | head -4
timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02d6_bench7.log 2>&1; bsum gpurun_out/r02d6_bench7.log
