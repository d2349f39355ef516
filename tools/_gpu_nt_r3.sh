mkdir -p gpurun_out
L=paper_2011_13579_b200/libvitertile_b200.so
cp $L /tmp/orig.so
: > gpurun_out/nt_r3_hash.txt
for v in def nt64 nt256; do
  cp libvariants/$v.so $L
  echo "== $v" >> gpurun_out/nt_r3_hash.txt
  timeout 300 python tools/bits_hash.py k7r3 26 >> gpurun_out/nt_r3_hash.txt 2>&1
done
cp /tmp/orig.so $L
timeout 600 python tools/code_bench.py k7r3 --log2n 28 --so libvariants/def.so,libvariants/nt64.so,libvariants/nt256.so > gpurun_out/nt_r3_ab.txt 2>&1
