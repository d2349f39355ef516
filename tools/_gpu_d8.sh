mkdir -p gpurun_out; OUT=gpurun_out/d8.txt; : > $OUT
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/d8_pytest.log 2>&1; echo "rc $?" >> gpurun_out/d8_pytest.log
LIB=paper_2011_13579_b200/libvitertile_b200.so; cp $LIB /tmp/lib_orig.so
for c in "k7r2 28" "k7r2 24" "k7r2 26" "k7r3 28" "k7r3 24"; do set -- $c; for v in nod8 d8s; do cp libvariants/$v.so $LIB; for r in 1 2; do echo -n "[$v] " >> $OUT; timeout 300 python tools/code_bench.py $1 --log2n $2 --one >> $OUT 2>&1; done; done; done
cp /tmp/lib_orig.so $LIB
