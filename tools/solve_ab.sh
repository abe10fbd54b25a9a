# solve-engine A/B (experiment; results in gpurun_out/ab.log)
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_v3.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_v3.log
for cfg in ${CFGS:-c2 c3 c4 c5}; do
 for v in "BLFLS_SOLVE_V3=0 BLFLS_FFT_V1=1" "BLFLS_V2_PASSES=0" "BLFLS_V2_PASSES=2 BLFLS_V2_PMAX_COLS=16" "BLFLS_V2_PASSES=2 BLFLS_V2_PMAX_COLS=32" "BLFLS_V2_PASSES=2 BLFLS_V2_PMAX_COLS=16 BLFLS_SOLVE_GROUP=0"; do
  echo "== $cfg $v" >> gpurun_out/ab.log
  env $v timeout 300 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'solve', round(d['roofline_solve']['frac'],3), round(d['roofline_solve']['ms_per_iter'],4), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/ab.log 2>&1
 done
done
