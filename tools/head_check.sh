# HEAD check: GPU tests, smoke, default bench line, reference arm, c2 launch list
out=gpurun_out/head
mkdir -p $out
timeout 1500 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
timeout 600 python bench.py > $out/bench_c2.log 2>&1
timeout 600 python bench.py --impl reference > $out/bench_reference_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch_c2.log 2>&1
