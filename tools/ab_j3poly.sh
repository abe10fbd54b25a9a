#!/bin/bash
# c5 shared-guide BLF: FMA-pipe exp2 of every k-th exponent pair (experiments build)
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/jp_default.json 2>&1
for k in 4 6 8 12 3; do BLFLS_LIBRARY=$EXP BLFLS_J3_POLY=$k $B > gpurun_out/jp_$k.json 2>&1; done
