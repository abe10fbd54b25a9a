#!/bin/bash
# c5 shared-guide BLF: row-block staging (default) vs per-cell staging (experiments build)
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/ab3_default.json 2>&1
BLFLS_LIBRARY=$EXP BLFLS_J3_STAGE=0 $B > gpurun_out/ab3_cell.json 2>&1
$B > gpurun_out/ab3_default2.json 2>&1
