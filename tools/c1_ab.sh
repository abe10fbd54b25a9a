# c1 (512^2, 1 iteration): solve engine A/B (results in gpurun_out/c1.log)
run() { echo "== $1 $2" >> gpurun_out/c1.log; env $2 timeout 300 python bench.py --config $1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/c1.log 2>&1; }
for v in "BLFLS_V2_PASSES=6" "BLFLS_V2_PASSES=0" "BLFLS_V2_PASSES=2" "BLFLS_V2_PASSES=4" "BLFLS_P2=1 BLFLS_V2_PASSES=0"; do run c1 "$v"; done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
