timeout 120 python -m pytest tests/test_gpu_clip_aggregate.py tests/test_gpu_kernels.py -q -x 2>&1 | tail -1
rm -f gpurun_out/r02n_aggmicro.log
for C in 100 1000 10000; do for impl in fused twopass; do
  timeout 300 python bench.py --workload aggmicro --cohort $C --micro-impl $impl --steps 5 --warmup 3 2>&1 | tail -1 >> gpurun_out/r02n_aggmicro.log
done; done
for Dm in 1000000 2000000 4000000; do for impl in fused twopass; do
  timeout 300 python bench.py --workload aggmicro --cohort 1000 --micro-dim $Dm --micro-impl $impl --steps 5 --warmup 3 2>&1 | tail -1 >> gpurun_out/r02n_aggmicro.log
done; done
python - <<'PY'
import json
for l in open('gpurun_out/r02n_aggmicro.log'):
    try: d = json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['config']['impl'], d['config']['D'], d['config']['cohort'], round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['frac'] for k, v in d['kernels'].items()})
PY
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"clip_aggregate_fused|noise_avg|row_sumsq|weighted_sum" -c 6 -o gpurun_out/r02n_agg python bench.py --workload aggmicro --cohort 64 --steps 1 --warmup 3 > gpurun_out/r02n_ncu.log 2>&1; echo ncu=$?
timeout 600 ncu --set full --clock-control none -k regex:"row_sumsq|weighted_sum" -c 2 -o gpurun_out/r02n_twopass python bench.py --workload aggmicro --cohort 64 --micro-impl twopass --steps 1 --warmup 3 > gpurun_out/r02n_ncu2.log 2>&1; echo ncu2=$?
