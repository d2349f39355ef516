mkdir -p gpurun_out
timeout 900 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/nt64.so,libvariants/nt64s1.so,libvariants/nt64s2.so,libvariants/nt64s3.so,libvariants/nt64s4.so,libvariants/nt64s5.so,libvariants/nt64s6.so > gpurun_out/nt64_seed.txt 2>&1
