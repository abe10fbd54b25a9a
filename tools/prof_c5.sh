# ncu --set full of the c5 shared-guide BLF kernel and the c5 column pass (one launch each)
out=gpurun_out/c5prof
mkdir -p $out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_blf_j3" -c 1 -o $out/j3_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_j3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_col" -c 1 -o $out/col_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_col.log 2>&1
ls -la $out
