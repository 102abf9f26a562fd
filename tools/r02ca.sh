set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02ca_pytest_gpu.log 2>&1; tail -3 gpurun_out/r02ca_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ca_smoke.log 2>&1; tail -2 gpurun_out/r02ca_smoke.log
timeout 600 python bench.py > gpurun_out/r02ca_bench.log 2>&1; tail -c 400 gpurun_out/r02ca_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02ca_ref.log 2>&1; tail -c 600 gpurun_out/r02ca_ref.log
