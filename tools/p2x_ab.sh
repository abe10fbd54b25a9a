# packed BLF tile height sweep (results in gpurun_out/p2x.log)
run() { echo "== $1 $2" >> gpurun_out/p2x.log; env $2 timeout 300 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), {k:round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> gpurun_out/p2x.log 2>&1; }
for cfg in c2 c4; do for t in 16 32; do run $cfg "BLFLS_P2_TH=$t"; done; done
for v in "BLFLS_P2=0" "BLFLS_P2=1 BLFLS_P2_TH=16" "BLFLS_P2=1 BLFLS_P2_TH=32" "BLFLS_P2=1 BLFLS_P2_TH=32 BLFLS_P2_POLY=10"; do run c3 "$v"; done
for v in "BLFLS_P2=0" "BLFLS_P2=1" "BLFLS_P2=1 BLFLS_P2_TH=8"; do run c1 "$v"; done
