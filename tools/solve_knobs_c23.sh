# A/B of the solve-pass knobs at the L2-resident configs c2 / c3 (stage times from the bench line)
out=gpurun_out/solve_c23
mkdir -p $out
for c in c2 c3; do
  for k in default BLFLS_V2_COLV=2 BLFLS_V2_PASSES=7 BLFLS_V2_ROWV=4 BLFLS_V2_ROWV=2 BLFLS_COL_PIPE=1 default; do
    if [ "$k" = default ]; then e=""; else e="$k"; fi
    env $e timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $out/${c}_${k}.log 2>&1
    tail -1 $out/${c}_${k}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms_per_step']; print('$c', '$k', round(d['value'],1), 'solve', round(d['roofline_solve']['frac'],3), {k: round(v,4) for k,v in s.items()})" >> $out/summary.txt 2>&1
  done
done
cat $out/summary.txt
