mkdir -p gpurun_out
LIB=paper_2011_13579_b200/libvitertile_b200.so
cp $LIB /tmp/lib_orig.so
cp libvariants/tmh2.so $LIB
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_large.py -q -x -m gpu -k "not K9 and not k9 and not K8 and not k8" > gpurun_out/tmh2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/tmh2_pytest.log
cp /tmp/lib_orig.so $LIB
: > gpurun_out/tmh2_ab.txt
for r in 1 2; do timeout 900 python tools/code_bench.py k7r2 --log2n 28 --so libvariants/def.so,libvariants/tmh2.so,libvariants/tmh2_s1.so,libvariants/tmh2_s2.so,libvariants/tmh2_s3.so >> gpurun_out/tmh2_ab.txt 2>&1; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum"
cp libvariants/tmh2.so $LIB
echo "[tmh2] ncu" >> gpurun_out/tmh2_ab.txt
timeout 300 ncu --metrics $M --clock-control none -k regex:vtk16 -s 2 -c 1 python tools/code_bench.py k7r2 --log2n 28 --one --steps 1 2>&1 | grep -E "dram__|gpu__time|lts__|inst_issued|inst_executed" >> gpurun_out/tmh2_ab.txt
cp /tmp/lib_orig.so $LIB
