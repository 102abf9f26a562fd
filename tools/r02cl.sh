bsum() { python - "$1" <<'PY'
import json,sys
d=[json.loads(x) for x in open(sys.argv[1]) if x.startswith("{")][-1]
print(d["value"], d["ms_per_step"]); print({k: round(v/d["profile_pass"]["steps"],3) for k,v in list(d["kernels_ms"].items())[:6]})
PY
}
timeout 300 python -m pytest tests/test_gpu_cnn.py -q -p no:warnings -x -k "cuda_core" > gpurun_out/r02cl_pytest.log 2>&1; tail -1 gpurun_out/r02cl_pytest.log
FB_CNN_CONV_IMPL=4 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02cl_bench128.log 2>&1; bsum gpurun_out/r02cl_bench128.log
touch paper_2404_06430_b200/csrc/cnn.cu; make -C paper_2404_06430_b200/csrc -j8 EXTRA_NVFLAGS=-DWF_CH=64 > /dev/null 2>&1; echo build=$?
FB_CNN_CONV_IMPL=4 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02cl_bench64.log 2>&1; bsum gpurun_out/r02cl_bench64.log
touch paper_2404_06430_b200/csrc/cnn.cu; make -C paper_2404_06430_b200/csrc -j8 EXTRA_NVFLAGS=-DWF_CH=256 > /dev/null 2>&1; echo build=$?
FB_CNN_CONV_IMPL=4 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/r02cl_bench256.log 2>&1; bsum gpurun_out/r02cl_bench256.log
