#!/bin/bash
# ncu --set full capture of the c5 shared-guide BLF kernel (8 images) + phase breakdown input
python tools/prof_blf_c5.py 8 && ncu --set full --clock-control none --import-source on -k regex:k_blf_j3r -c 1 -o gpurun_out/r02_ncu_blf_c5_j3r -f python tools/prof_blf_c5.py 8 > gpurun_out/j3r_ncu.log 2>&1
ncu -i gpurun_out/r02_ncu_blf_c5_j3r.ncu-rep --page raw --csv > gpurun_out/r02_ncu_blf_c5_j3r.csv
ncu -i gpurun_out/r02_ncu_blf_c5_j3r.ncu-rep --page source --csv > gpurun_out/r02_ncu_blf_c5_j3r_source.csv
tail -2 gpurun_out/j3r_ncu.log
