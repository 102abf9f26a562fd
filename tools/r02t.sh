timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02t_pytest_gpu.log 2>&1; tail -4 gpurun_out/r02t_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
for C in 1000 10000; do
  timeout 300 python bench.py --workload aggmicro --cohort $C --steps 5 --warmup 3 2>&1 | tail -1 >> gpurun_out/r02t_aggmicro.log
done
python - <<'PY'
import json
for l in open('gpurun_out/r02t_aggmicro.log'):
    d = json.loads(l); print(d['config']['impl'], d['config']['pool'], d['config']['cohort'], round(d['ms_per_step'],3), d['roofline']['frac'], {k: v['frac'] for k, v in d['kernels'].items()})
PY
