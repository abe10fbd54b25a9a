#!/bin/bash
# row-FFT shared-memory padding: one slot per 8 (default) vs per 16 (-DBLFLS_ROWPAD16 experiments build)
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
for c in c5 c2 c3 c4; do
  B="python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
  $B > gpurun_out/rp_${c}_8.json 2>&1
  BLFLS_LIBRARY=$EXP $B > gpurun_out/rp_${c}_16.json 2>&1
done
