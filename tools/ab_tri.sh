#!/bin/bash
# column pass A/B: cyclic tridiagonal solve (k_col_tri) shapes vs the column FFT pair
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
O=gpurun_out/tri_ab.txt
: > $O
run() { echo "## $*" >> $O; env BLFLS_LIBRARY=$EXP "$@" >> $O 2>&1; }
for shape in "2048 2048 3 64" "1024 1024 3 1" "1080 1920 3 1" "4096 4096 1 1" "512 512 1 1"; do
  run BLFLS_COL_TRI=0 python tools/solve_bench.py $shape 20
  for rpt in 32 16 8; do
    for sh in 0 1 2 3; do
      run BLFLS_TRI_RPT=$rpt BLFLS_TRI_SHAPE=$sh python tools/solve_bench.py $shape 20
    done
  done
done
