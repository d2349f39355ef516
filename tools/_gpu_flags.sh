mkdir -p gpurun_out
L=paper_2011_13579_b200/libvitertile_b200.so
cp $L /tmp/orig.so
: > gpurun_out/flags_hash.txt
for v in def o1; do
  cp libvariants/$v.so $L
  echo "== $v" >> gpurun_out/flags_hash.txt
  timeout 300 python tools/bits_hash.py k7r2 26 >> gpurun_out/flags_hash.txt 2>&1
done
cp /tmp/orig.so $L
timeout 600 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/o1.so,libvariants/o2.so > gpurun_out/flags_ab.txt 2>&1
timeout 600 python tools/code_bench.py k7r3 --log2n 28 --so libvariants/def.so,libvariants/o1.so > gpurun_out/flags_ab_r3.txt 2>&1
timeout 600 python tools/code_bench.py k9r2 --log2n 28 --so libvariants/def.so,libvariants/o1.so > gpurun_out/flags_ab_k9.txt 2>&1
