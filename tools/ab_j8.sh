#!/bin/bash
# A/B of the c5 shared-guide BLF kernels (experiments build)
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
for cfg in "BLFLS_J8=0" "BLFLS_J8=1" "BLFLS_J8=1 BLFLS_J8_POLY=4" "BLFLS_J8=1 BLFLS_J8_POLY=6" "BLFLS_J8=1 BLFLS_J8_POLY=8" "BLFLS_J8=1 BLFLS_J8_POLY=12" "BLFLS_J8=1 BLFLS_J8_TH=24" "BLFLS_J8=1 BLFLS_J8_TH=24 BLFLS_J8_POLY=6"; do
  name=$(echo $cfg | tr ' =' '_-')
  env $cfg BLFLS_LIBRARY=$EXP $B > gpurun_out/ab2_$name.json 2>&1
done
