#!/bin/bash
EXP=paper_1812_07122_b200/_lib_exp/libblfls.so
python tools/prof_blf_c5.py > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_blf_j -s 1 -c 1 -o gpurun_out/prof_j8 python tools/prof_blf_c5.py > gpurun_out/ncu_j8.log 2>&1
BLFLS_LIBRARY=$EXP BLFLS_J8=0 python tools/prof_blf_c5.py > gpurun_out/prof_plain3.log 2>&1 && \
BLFLS_LIBRARY=$EXP BLFLS_J8=0 ncu --set full --clock-control none --import-source on -k regex:k_blf_j -s 1 -c 1 -o gpurun_out/prof_j3 python tools/prof_blf_c5.py > gpurun_out/ncu_j3.log 2>&1
echo done
