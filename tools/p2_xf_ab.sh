# A/B of the factorised-exponent self-guided kernel: geometry (BLFLS_P2_XFG) and exp2 period
out=gpurun_out/p2xf
mkdir -p $out
run() { env "$@" timeout 300 python bench.py --config $C --steps 3 --no-cpu-baseline --no-e2e > $out/tmp.log 2>&1; tail -1 $out/tmp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', '$*', round(d['value'],1), round(d['roofline']['frac'],4))" >> $out/summary.txt; }
for C in c2 c4; do
  run BLFLS_P2_XF=0
  for g in 0 1 2; do run BLFLS_P2_XF=1 BLFLS_P2_XFG=$g; done
  for k in 5 6 8; do for g in 0 1 2; do run BLFLS_P2_XF=1 BLFLS_P2_XFG=$g BLFLS_P2_POLY=$k; done; done
done
cat $out/summary.txt
