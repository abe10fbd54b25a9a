# round-end evidence: GPU tests, smoke, all-config bench lines, reference arm, launch lists (c1, c2, c3)
out=gpurun_out/final
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for c in c1 c2 c3 c4 c5; do timeout 600 python bench.py --config $c > $out/bench_$c.log 2>&1; done
timeout 300 python bench.py --impl reference > $out/bench_reference_c2.log 2>&1
for c in c1 c2 c3; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch_$c.log 2>&1
done
du -sh gpurun_out
