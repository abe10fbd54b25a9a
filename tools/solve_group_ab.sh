# c5 solve: plane-group size x FFT engine (experiment; results in gpurun_out/group.log)
for v in "BLFLS_FFT_V1=1" "BLFLS_V2_PMAX_ROWS=16 BLFLS_V2_PMAX_COLS=16"; do
 for g in 1 2 4 8 0; do
  echo "== c5 group=$g $v" >> gpurun_out/group.log
  env $v BLFLS_SOLVE_GROUP=$g timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], 'solve', d['roofline_solve']['frac'], d['roofline_solve']['ms_per_iter'])" >> gpurun_out/group.log 2>&1
 done
done
