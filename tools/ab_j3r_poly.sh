#!/bin/bash
# c5 two-row shared-guide BLF: FMA-pipe exp2 of every k-th exponent pair (experiments build)
E=paper_1812_07122_b200/_lib_exp/libblfls.so
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
for k in 0 24 16 12 10 8 6; do
  BLFLS_LIBRARY=$E BLFLS_J3R_POLY=$k $B > gpurun_out/j3r_poly_$k.json 2>&1
  python -c "
import json,sys
d=json.loads(open('gpurun_out/j3r_poly_$k.json').read().strip().splitlines()[-1]); print('poly', $k, round(d['value']), round(d['roofline']['frac'],4), round(d['stage_ms_per_step']['grad_blf'],2))"
done
