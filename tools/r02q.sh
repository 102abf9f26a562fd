timeout 900 python -m pytest tests/test_gpu_lm.py -q -x -p no:warnings 2>&1 | tail -30
