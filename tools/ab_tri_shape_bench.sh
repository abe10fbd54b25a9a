#!/bin/bash
# column pass thread shape / rows per thread measured by the bench's stage timers (cold L2 between steps)
E=paper_1812_07122_b200/_lib_exp/libblfls.so
for c in c1 c2 c3 c4 c5; do for rpt in 32 16; do for sh in 0 1 2; do
  BLFLS_LIBRARY=$E BLFLS_TRI_RPT=$rpt BLFLS_TRI_SHAPE=$sh python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ts.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/ts.json')); print('$c rpt $rpt shape $sh', round(d['value'],1), 'col', round(d['stage_ms_per_step']['col_solve'],4))"
done; done; done
