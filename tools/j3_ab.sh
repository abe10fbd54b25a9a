# shared-guide BLF variants on c5 (results in gpurun_out/j3.log)
run() { echo "== $1 $2" >> gpurun_out/j3.log; env $2 timeout 300 python bench.py --config $1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), 'solve', round(d['roofline_solve']['frac'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/j3.log 2>&1; }
for v in "BLFLS_J3X=0" "BLFLS_J3X=2" "BLFLS_J3X=3"; do run c5 "$v"; done
