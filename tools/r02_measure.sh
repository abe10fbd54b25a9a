#!/bin/bash
# round-2 measurement set: every config's bench line, the c5 launch list
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 10 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err; done
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_c5_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_launch.log 2>&1
echo done
