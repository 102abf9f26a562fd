set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02cv_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02cv_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02cv_smoke.log 2>&1; tail -2 gpurun_out/r02cv_smoke.log
timeout 600 python bench.py > gpurun_out/r02cv_bench.log 2>&1; tail -c 300 gpurun_out/r02cv_bench.log
timeout 600 python bench.py --workload aggmicro > gpurun_out/r02cv_aggmicro.log 2>&1; tail -c 400 gpurun_out/r02cv_aggmicro.log
