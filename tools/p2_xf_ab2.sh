# focused A/B (5 timed steps, clocks reported): difference form vs factorised exponents
out=gpurun_out/p2xf2
mkdir -p $out
run() { env "$@" timeout 300 python bench.py --config $C --steps 5 --no-cpu-baseline --no-e2e > $out/tmp.log 2>&1; tail -1 $out/tmp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', '$*', round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['frac'],4), round(d['stage_ms_per_step']['grad_blf'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" >> $out/summary.txt; }
for rep in 1 2; do
C=c2; run BLFLS_P2_XF=0; run BLFLS_P2_XF=1 BLFLS_P2_POLY=6; run BLFLS_P2_XF=1 BLFLS_P2_POLY=7
C=c4; run BLFLS_P2_XF=0; run BLFLS_P2_XF=1 BLFLS_P2_POLY=5; run BLFLS_P2_XF=1 BLFLS_P2_POLY=6
done
cat $out/summary.txt
