mkdir -p gpurun_out
: > gpurun_out/ab3.txt
for r in 1 2; do
  timeout 900 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/pf75.so,libvariants/pf50.so,libvariants/ef0.so >> gpurun_out/ab3.txt 2>&1
  timeout 900 python tools/code_bench.py k9r2 --log2n 28 --so libvariants/def.so,libvariants/mc0.so,libvariants/mbf16.so,libvariants/mbf48.so >> gpurun_out/ab3.txt 2>&1
  timeout 900 python tools/code_bench.py k8r2 --log2n 28 --so libvariants/def.so,libvariants/mc0.so,libvariants/mbf16.so,libvariants/mbf48.so >> gpurun_out/ab3.txt 2>&1
done
