E=paper_1812_07122_b200/_lib_exp/libblfls.so
for t in 200 95 85 50; do for shape in "1080 1920 3 1" "1024 1024 3 1" "2048 2048 3 64"; do echo "comp>$t% $shape: $(BLFLS_LIBRARY=$E BLFLS_TRI_COMP=$t python tools/solve_bench.py $shape 20)"; done; done
