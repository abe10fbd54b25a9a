# ncu --set full of the c2 column pass (auto-pipelined) and the plain pass for comparison
out=gpurun_out/colprof
mkdir -p $out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_col" -c 1 -o $out/colpipe_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_pipe.log 2>&1
BLFLS_COL_PIPE=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_col" -c 1 -o $out/colplain_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_plain.log 2>&1
ls -la $out
