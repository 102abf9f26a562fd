#!/bin/bash
# ResNet-18 (config D) first GPU run: parity tests
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_resnet.py -q -p no:warnings -x --timeout 600 > gpurun_out/r02ae_pytest.log 2>&1
tail -30 gpurun_out/r02ae_pytest.log
