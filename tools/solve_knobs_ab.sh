# A/B of the solve-pass knobs (column vectors per CTA, row r2c engine) at c2 / c5
out=gpurun_out/solve_ab
mkdir -p $out
for c in c5 c2 c4; do
  for k in "default" "BLFLS_V2_COLV=2" "BLFLS_V2_PASSES=7" "BLFLS_V2_COLV=8"; do
    if [ "$k" = default ]; then e=""; else e="$k"; fi
    env $e timeout 300 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e > $out/${c}_${k}.log 2>&1
    tail -1 $out/${c}_${k}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms_per_step']; print('$c', '$k', round(d['value'],1), 'solve', round(d['roofline_solve']['frac'],3), {k: round(v,3) for k,v in s.items()})" >> $out/summary.txt
  done
done
cat $out/summary.txt
