set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02d5_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02d5_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d5_smoke.log 2>&1; tail -2 gpurun_out/r02d5_smoke.log
timeout 600 python bench.py > gpurun_out/r02d5_bench.log 2>&1; tail -c 300 gpurun_out/r02d5_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/r02d5_launches.csv python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline --profile-steps 1 > gpurun_out/r02d5_ncu.log 2>&1; echo ncu=$?
