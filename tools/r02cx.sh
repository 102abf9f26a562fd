agg() { for C in 100 1000 10000; do timeout 600 python bench.py --workload aggmicro --cohort $C > gpurun_out/r02cx_agg_$1_$C.log 2>&1; grep '^{' gpurun_out/r02cx_agg_$1_$C.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', $C, d['value'], d['roofline']['frac'], {k: v['frac'] for k,v in d['kernels'].items()})"; done; }
timeout 600 python -m pytest tests/test_gpu_clip_aggregate.py -q -p no:warnings > gpurun_out/r02cx_pytest.log 2>&1; tail -1 gpurun_out/r02cx_pytest.log
agg nofence
touch paper_2404_06430_b200/csrc/clip_aggregate_fused.cu; make -C paper_2404_06430_b200/csrc -j8 EXTRA_NVFLAGS=-DFB_RING_PROXY_FENCE > /dev/null 2>&1; echo build=$?
agg fence
