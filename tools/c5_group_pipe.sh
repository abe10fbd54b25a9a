# c5 solve: plane-group size with the auto-selected (L2-resident => pipelined) column pass
out=gpurun_out/c5grp
mkdir -p $out
for k in "BLFLS_SOLVE_GROUP=0" "BLFLS_SOLVE_GROUP=1" "BLFLS_SOLVE_GROUP=2" "BLFLS_SOLVE_GROUP=2 BLFLS_COL_PIPE=0" "BLFLS_SOLVE_GROUP=1 BLFLS_COL_PIPE=0" "X=default"; do
  env $k timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $out/log 2>&1
  tail -1 $out/log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms_per_step']; print('$k', round(d['value'],1), 'solve', round(d['roofline_solve']['frac'],3), d['roofline_solve']['ms_per_iter'], {k: round(v,3) for k,v in s.items()})" >> $out/summary.txt 2>&1
done
cat $out/summary.txt
