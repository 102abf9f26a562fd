timeout 300 python -m pytest tests/test_gpu_clip_aggregate.py -q -p no:warnings 2>&1 | tail -2
rm -f gpurun_out/r02w_aggmicro.log
for C in 100 1000 10000; do
  timeout 300 python bench.py --workload aggmicro --cohort $C --steps 5 --warmup 3 2>&1 | tail -1 >> gpurun_out/r02w_aggmicro.log
done
python - <<'PY'
import json
for l in open('gpurun_out/r02w_aggmicro.log'):
    d = json.loads(l); print(d['config']['impl'], d['config']['cohort'], round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['frac'] for k, v in d['kernels'].items()})
PY
