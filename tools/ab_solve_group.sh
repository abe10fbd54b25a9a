#!/bin/bash
# c5 solve: plane groups (spectrum L2-resident across r2c -> column -> c2r, two streams) vs one launch per pass
E=paper_1812_07122_b200/_lib_exp/libblfls.so
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline"
for g in 0 3 6 9 12 24 48; do
  BLFLS_LIBRARY=$E BLFLS_SOLVE_GROUP=$g $B > gpurun_out/sg_$g.json 2>&1
  python -c "
import json
d=json.loads(open('gpurun_out/sg_$g.json').read().strip().splitlines()[-1]); s=d['stage_ms_per_step']; print('group', $g, round(d['value']), round(d['ms_per_step'],2), {k:round(v,2) for k,v in s.items()})"
done
