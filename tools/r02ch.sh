bsum() { python - "$1" <<'PY'
import json,sys
d=[json.loads(x) for x in open(sys.argv[1]) if x.startswith("{")][-1]
print(d["value"], d["ms_per_step"]); print({k: round(v/d["profile_pass"]["steps"],3) for k,v in list(d["kernels_ms"].items())[:8]})
PY
}
FB_CNN_CONV_IMPL=4 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02ch_bench4.log 2>&1; bsum gpurun_out/r02ch_bench4.log
grep conv1_bwd gpurun_out/r02ch_bench4.log | head -2 | cut -c1-300
