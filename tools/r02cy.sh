agg() { for C in 100 1000; do timeout 600 python bench.py --workload aggmicro --cohort $C > gpurun_out/r02cy_agg_$1_$C.log 2>&1; grep '^{' gpurun_out/r02cy_agg_$1_$C.log | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', $C, d['value'], d['roofline']['frac'], {k: v['frac'] for k,v in d['kernels'].items()})"; done; }
agg cur
cp scratch/old_caf.cu paper_2404_06430_b200/csrc/clip_aggregate_fused.cu; make -C paper_2404_06430_b200/csrc -j8 > gpurun_out/r02cy_build.log 2>&1; echo build=$?
agg old
