mkdir -p gpurun_out
timeout 1200 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/s25.so,libvariants/s26.so,libvariants/s27.so,libvariants/s28.so,libvariants/s29.so,libvariants/s30.so,libvariants/s31.so,libvariants/s32.so > gpurun_out/seed3.txt 2>&1
