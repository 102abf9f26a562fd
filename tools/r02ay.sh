#!/bin/bash
# memcheck over the new GEMM epilogue; ncu on a small LM test
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_lm.py tests/test_gpu_resnet.py -q -p no:warnings -x -k "(tcgen05 and (mid or tiny or wide32 or narrow)) or deterministic" > gpurun_out/r02ay_memcheck.log 2>&1; echo memcheck=$?; tail -3 gpurun_out/r02ay_memcheck.log
unset PYTORCH_NO_CUDA_MEMORY_CACHING
timeout 600 ncu --metrics gpu__time_duration.sum,sm__ops_path_tensor_src_tf32_dst_fp32.sum --clock-control none -k regex:"gemm_tc_kernel" -c 5 python -m pytest tests/test_gpu_lm.py -q -p no:warnings -x -k "tcgen05 and 1-16-0.3-0.0-mid" > gpurun_out/r02ay_ncu.log 2>&1; echo ncu=$?; grep -E "ERROR|passed|failed" gpurun_out/r02ay_ncu.log | head -5
