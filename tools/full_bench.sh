# all-config bench lines, reference arm, c2 launch list, ncu captures of the dominant kernels
# (outputs in gpurun_out/full; summarised under profiles/; keep the total under gpurun's 64 MiB)
out=gpurun_out/full
mkdir -p $out
for c in c1 c2 c3 c4 c5; do timeout 600 python bench.py --config $c > $out/bench_$c.log 2>&1; done
timeout 300 python bench.py --impl reference > $out/bench_reference_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_blf_p2" -c 1 -o $out/blf_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c2.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size,launch__block_size,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_blf_p2" -c 1 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c4.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_blf_j3" -c 1 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_c5.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_row_r2c|k2_col|k2_row_c2r|k_col|k_row_c2r" -c 3 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_solve_c2.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_row_r2c|k2_col|k2_row_c2r|k_col|k_row_c2r" -c 3 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_solve_c5.csv 2>&1
du -sh gpurun_out
