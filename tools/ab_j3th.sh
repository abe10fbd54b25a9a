#!/bin/bash
# c5 shared-guide BLF: 32-row (default since r02) vs 16-row tiles (experiments build)
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/th_32.json 2>&1
BLFLS_LIBRARY=$EXP BLFLS_J3_TH=16 $B > gpurun_out/th_16.json 2>&1
