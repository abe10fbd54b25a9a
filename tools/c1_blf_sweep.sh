# c1 (512^2 gray, r = 5, one partial wave): tile rows x FMA-pipe exp2 period of the packed BLF
out=gpurun_out/c1sweep
mkdir -p $out
for k in X=default BLFLS_P2_TH=16 BLFLS_P2_TH=32 BLFLS_P2_POLY=0 "BLFLS_P2_TH=16 BLFLS_P2_POLY=0" BLFLS_P2_POLY=8 X=default; do
  env $k timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $out/log 2>&1
  tail -1 $out/log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', round(d['value'],1), round(d['ms_per_step'],4), 'blf', round(d['roofline']['frac'],3), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> $out/summary.txt 2>&1
done
cat $out/summary.txt
