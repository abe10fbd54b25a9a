#!/bin/bash
# round-2 evidence set (1 x B200): GPU tests, smoke, the driver's bench lines, torchrun N=1,
# the reference arm, the c5 launch list and ncu --set full captures of the two new kernels
O=gpurun_out
python -m pytest tests -q -m gpu > $O/final_pytest.txt 2>&1; echo rc=$? >> $O/final_pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.txt 2>&1; echo rc=$? >> $O/final_smoke.txt
python bench.py --steps 20 --warmup 5 > $O/final_c5.json 2> $O/final_c5.err
for c in c1 c2 c3 c4; do python bench.py --config $c --steps 20 --warmup 5 > $O/final_$c.json 2> $O/final_$c.err; done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 5 --warmup 3 > $O/final_torchrun1.json 2> $O/final_torchrun1.err
python bench.py --impl reference --steps 20 --warmup 5 > $O/final_ref.json 2> $O/final_ref.err
python tools/parity_report.py > $O/final_parity.txt 2>&1
# launch list of the bench command (after it ran clean above)
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-other-configs > $O/final_c5_short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_c5.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-other-configs > $O/final_ncu_launch.log 2>&1
# --set full of the 64-image BLF launch and of the column pass (24 planes)
python tools/prof_blf_c5.py 64 > $O/final_prof_blf.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blf_j3r -c 1 -o $O/r02_ncu_blf_c5_j3r -f \
    python tools/prof_blf_c5.py 64 > $O/final_ncu_blf.log 2>&1
ncu -i $O/r02_ncu_blf_c5_j3r.ncu-rep --page raw --csv > $O/r02_ncu_blf_c5_j3r.csv 2>/dev/null
ncu -i $O/r02_ncu_blf_c5_j3r.ncu-rep --page source --csv > $O/r02_ncu_blf_c5_j3r_source.csv 2>/dev/null
python tools/prof_solve_c5.py 8 > $O/final_prof_solve.txt 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_col_tri|k_row_r2c|k2_row_c2r" -c 3 -o $O/r02_ncu_solve_c5 -f \
    python tools/prof_solve_c5.py 8 > $O/final_ncu_solve.log 2>&1
ncu -i $O/r02_ncu_solve_c5.ncu-rep --page raw --csv > $O/r02_ncu_solve_c5.csv 2>/dev/null
echo done
