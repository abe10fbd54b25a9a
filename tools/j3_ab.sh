# packed shared-guide BLF A/B (experiment; results in gpurun_out/j3.log)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_j3.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_j3.log
for v in "BLFLS_J3=0" "BLFLS_J3_MINB=4" "BLFLS_J3_MINB=3"; do
  echo "== c5 $v" >> gpurun_out/j3.log
  env $v timeout 300 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), 'solve', round(d['roofline_solve']['frac'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/j3.log 2>&1
done
