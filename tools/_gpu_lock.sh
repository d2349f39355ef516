mkdir -p gpurun_out
L=paper_2011_13579_b200/libvitertile_b200.so
cp $L /tmp/orig.so
: > gpurun_out/lock_hash.txt
for v in def nt256 lock1 lock2; do
  cp libvariants/$v.so $L
  echo "== $v" >> gpurun_out/lock_hash.txt
  timeout 300 python tools/bits_hash.py k7r2 26 >> gpurun_out/lock_hash.txt 2>&1
done
cp /tmp/orig.so $L
: > gpurun_out/lock_ab.txt
for r in 1 2; do
  timeout 900 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/nt256.so,libvariants/lock1.so,libvariants/lock2.so >> gpurun_out/lock_ab.txt 2>&1
done
