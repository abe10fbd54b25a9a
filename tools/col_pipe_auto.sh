# the auto-selected pipelined column pass: GPU tests, then c2 / c4 A/B against the plain pass
out=gpurun_out/colauto
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
for c in c2 c4; do
  for k in auto BLFLS_COL_PIPE=0 auto BLFLS_COL_PIPE=0; do
    if [ "$k" = auto ]; then e=""; else e="$k"; fi
    env $e timeout 300 python bench.py --config $c --steps 10 --no-cpu-baseline --no-e2e > $out/${c}_${k}.log 2>&1
    tail -1 $out/${c}_${k}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stage_ms_per_step']; print('$c', '$k', round(d['value'],1), 'solve', round(d['roofline_solve']['frac'],3), {k: round(v,4) for k,v in s.items()})" >> $out/summary.txt 2>&1
  done
done
timeout 300 python bench.py > $out/bench_default.log 2>&1
cat $out/summary.txt; tail -n 2 $out/pytest_gpu.log
