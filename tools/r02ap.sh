#!/bin/bash
# ResNet: parity after the GN / permute rework, full bench line (with the host-CPU port
# baseline, one client), and an ncu capture of the grouped-GEMM launches
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -s --timeout 900 > gpurun_out/r02ap_pytest.log 2>&1
tail -2 gpurun_out/r02ap_pytest.log
timeout 1200 python bench.py --workload resnet --steps 5 --warmup 3 --e2e-steps 2 --e2e-warmup 20 --profile-steps 2 > gpurun_out/r02ap_bench.log 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/r02ap_bench.log") if x.startswith("{")]
d=json.loads(l[-1]); print(d["value"], d["ms_per_step"], d.get("e2e"), d.get("cpu_baseline")); print({k: round(v/d["profile_pass"]["steps"],1) for k,v in list(d["kernels_ms"].items())[:12]})
PY
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__ops_path_tensor_src_tf32_dst_fp32.sum,smsp__sass_inst_executed_op_utcmma.sum,l1tex__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size --clock-control none -k regex:"gemm_tc_kernel" -s 600 -c 60 --csv python bench.py --workload resnet --steps 1 --warmup 3 --e2e-steps 0 --profile-steps 1 --no-cpu-baseline > gpurun_out/r02ap_ncu.csv 2> gpurun_out/r02ap_ncu.err
tail -1 gpurun_out/r02ap_ncu.err; wc -l gpurun_out/r02ap_ncu.csv
