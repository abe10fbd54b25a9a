# ncu of the packed self-guided kernel at c2 (r = 7) with and without FMA-pipe exp2 offload
for pp in 0 7; do
BLFLS_P2=1 BLFLS_P2_POLY=$pp ncu --set full --clock-control none -k regex:"k_blf_p2" -c 1 -o gpurun_out/p2_c2_poly$pp python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p2_$pp.log 2>&1
done
ncu --set full --clock-control none -k regex:"k_grad_blf" -c 1 -o gpurun_out/blf_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_blf.log 2>&1
