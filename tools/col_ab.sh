# column pass: k_col (v1) vs the high-radix k2_col capped at 64 registers (results in gpurun_out/col.log)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_col.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_col.log
for cfg in c2 c3 c4 c5; do
 for v in "BLFLS_V2_PASSES=4" "BLFLS_V2_PASSES=6"; do
  echo "== $cfg $v" >> gpurun_out/col.log
  env $v timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), 'solve', round(d['roofline_solve']['frac'],3), round(d['roofline_solve']['ms_per_iter'],4), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/col.log 2>&1
 done
done
for s in "2048 2048 3 16"; do
 for v in "BLFLS_V2_PASSES=4" "BLFLS_V2_PASSES=6"; do
  echo "$s $v: $(env BLFLS_SOLVE_GROUP=0 $v python tools/solve_bench.py $s 20)" >> gpurun_out/col.log
 done
done
