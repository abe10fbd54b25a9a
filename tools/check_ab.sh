# tests + bench of c1..c4 with the current defaults (results in gpurun_out/check.log)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_check.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_check.log
run() { echo "== $1 $2" >> gpurun_out/check.log; env $2 timeout 300 python bench.py --config $1 --steps ${3:-5} --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), 'solve', round(d['roofline_solve']['frac'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/check.log 2>&1; }
run c1 "" 20; run c2 ""; run c3 ""; run c3 "BLFLS_P2=0"; run c4 ""
