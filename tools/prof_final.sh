# ncu --set full of the DEFAULT BLF kernel at c2 / c4 / c5 (one launch each) at HEAD, for the traffic figures
out=gpurun_out/proffinal
mkdir -p $out
for c in c2 c4 c5; do
  k="k_blf_p2"; [ $c = c5 ] && k="k_blf_j3"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o $out/blf_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_$c.log 2>&1
  echo "$c rc=$?" >> $out/rc.txt
done
ls -la $out
