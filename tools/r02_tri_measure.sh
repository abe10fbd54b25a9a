#!/bin/bash
# tridiagonal column pass: GPU tests, c5 bench line, ncu capture of the pass, launch list
python -m pytest tests -x -q -m gpu > gpurun_out/tri_pytest_all.txt 2>&1; echo rc=$? >> gpurun_out/tri_pytest_all.txt
python bench.py --steps 20 --warmup 5 > gpurun_out/tri_c5.json 2> gpurun_out/tri_c5.err
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/tri_$c.json 2> gpurun_out/tri_$c.err; done
python tools/prof_solve_c5.py 8 > gpurun_out/tri_prof_plain.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_col_tri -c 1 -o gpurun_out/r02_ncu_col_tri_c5 -f \
    python tools/prof_solve_c5.py 8 > gpurun_out/tri_ncu.log 2>&1
ncu -i gpurun_out/r02_ncu_col_tri_c5.ncu-rep --page raw --csv > gpurun_out/r02_ncu_col_tri_c5.csv 2>/dev/null
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/tri_c5_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5_tri.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/tri_ncu_launch.log 2>&1
echo done
