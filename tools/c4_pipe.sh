# c4 (4096-point columns, one plane): pipelined vs plain column pass
out=gpurun_out/c4pipe
mkdir -p $out
for k in BLFLS_COL_PIPE=1 BLFLS_COL_PIPE=0 BLFLS_COL_PIPE=1 BLFLS_COL_PIPE=0; do
  env $k timeout 300 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $out/log 2>&1
  tail -1 $out/log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$k', round(d['value'],1), 'solve', round(d['roofline_solve']['frac'],3), {k: round(v,4) for k,v in d['stage_ms_per_step'].items()})" >> $out/summary.txt 2>&1
done
cat $out/summary.txt
