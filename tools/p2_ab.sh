# packed BLF kernels A/B (experiment; results in gpurun_out/p2.log)
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_p2.log 2>&1; echo pytest_exit=$? >> gpurun_out/pytest_p2.log
run() { echo "== $1 $2" >> gpurun_out/p2.log; env $2 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), 'solve', round(d['roofline_solve']['frac'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/p2.log 2>&1; }
for cfg in c2 c3; do for v in "BLFLS_P2=0" "BLFLS_P2=1 BLFLS_P2_POLY=0" "BLFLS_P2=1 BLFLS_P2_POLY=7" "BLFLS_P2=1 BLFLS_P2_POLY=5"; do run $cfg "$v"; done; done
for v in "BLFLS_P2=0" "BLFLS_P2_POLY=7" "BLFLS_P2_POLY=5"; do run c4 "$v"; done
run c5 "BLFLS_J3=1"
