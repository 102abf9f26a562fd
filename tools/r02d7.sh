timeout 1500 python -m pytest tests -m gpu -q -p no:warnings > gpurun_out/r02d7_pytest_gpu.log 2>&1; tail -2 gpurun_out/r02d7_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d7_smoke.log 2>&1; tail -2 gpurun_out/r02d7_smoke.log
