# solve kernels in the streaming regime (48 planes of 2048^2, one launch per pass)
export BLFLS_SOLVE_GROUP=0 BLFLS_SOLVE_V3=0
for pm in 32 16; do
BLFLS_V2_PMAX_ROWS=$pm BLFLS_V2_PMAX_COLS=$pm python tools/solve_bench.py 2048 2048 3 16 >> gpurun_out/sb.log 2>&1
BLFLS_V2_PMAX_ROWS=$pm BLFLS_V2_PMAX_COLS=$pm ncu --set full --clock-control none -k regex:"k2_" -c 3 -o gpurun_out/v2_${pm}_solve python tools/solve_bench.py 2048 2048 3 16 1 > gpurun_out/ncu2_$pm.log 2>&1
done
for s in "1024 1024 3 1" "1080 1920 3 1" "4096 4096 1 1" "2048 2048 3 16"; do
 for v in "BLFLS_FFT_V1=1" "BLFLS_V2_PMAX_ROWS=32 BLFLS_V2_PMAX_COLS=32" "BLFLS_V2_PMAX_ROWS=16 BLFLS_V2_PMAX_COLS=16"; do
  echo "$s $v: $(env $v python tools/solve_bench.py $s 20)" >> gpurun_out/sb2.log
 done
done
