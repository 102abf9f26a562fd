#!/bin/bash
# 16-row epilogue tiles: LM + ResNet parity, both benches, then the ncu GEMM capture
bash tools/r02av.sh
bash tools/r02ax.sh
grep -c "gemm_tc" gpurun_out/r02ax_lm_ncu.csv gpurun_out/r02ax_rn_ncu.csv
