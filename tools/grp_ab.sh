# c5 solve plane-group sweep + c2 default check (results in gpurun_out/grp.log)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_grp.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_grp.log
run() { echo "== $1 $2" >> gpurun_out/grp.log; env $2 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), 'solve', round(d['roofline_solve']['frac'],3), round(d['roofline_solve']['ms_per_iter'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/grp.log 2>&1; }
run c2 ""
for g in 1 2 3 4 6 0; do run c5 "BLFLS_SOLVE_GROUP=$g"; done
