mkdir -p gpurun_out
L=paper_2011_13579_b200/libvitertile_b200.so
cp $L /tmp/orig.so
: > gpurun_out/nt64_hash.txt
for v in def nt64; do
  cp libvariants/$v.so $L
  echo "== $v" >> gpurun_out/nt64_hash.txt
  timeout 300 python tools/bits_hash.py k7r2 26 >> gpurun_out/nt64_hash.txt 2>&1
done
cp /tmp/orig.so $L
timeout 600 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/nt64.so > gpurun_out/nt64_ab.txt 2>&1
timeout 600 python tools/code_bench.py k7r2 --log2n 24 --so libvariants/def.so,libvariants/nt64.so >> gpurun_out/nt64_ab.txt 2>&1
