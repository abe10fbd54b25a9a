#!/bin/bash
# c3 self-guided BLF (sigma_r = 0.05: difference form): two rows per thread (k_blf_p2r<5, .., XF = false>) vs k_blf_p2
E=paper_1812_07122_b200/_lib_exp/libblfls.so
for v in "BLFLS_P2R_DIFF=0" "BLFLS_P2R_POLY=0" "BLFLS_P2R_POLY=12" "BLFLS_P2R_POLY=8" "BLFLS_P2R_POLY=6" "BLFLS_P2R_POLY=5" "BLFLS_P2R_POLY=4" "BLFLS_P2R_POLY=3"; do
  env BLFLS_LIBRARY=$E $v python bench.py --config c3 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p2r.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/p2r.json')); print('c3 $v', round(d['value'],1), round(d['roofline']['frac'],4), round(d['stage_ms_per_step']['grad_blf'],4))"
done
