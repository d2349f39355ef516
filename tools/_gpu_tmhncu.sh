mkdir -p gpurun_out
LIB=paper_2011_13579_b200/libvitertile_b200.so
cp $LIB /tmp/lib_orig.so
cp libvariants/tmh.so $LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vtk16 -s 2 -c 1 -f -o gpurun_out/r2_k16tmh python tools/code_bench.py k7r2 --log2n 28 --one --steps 1 > /dev/null 2>&1
cp /tmp/lib_orig.so $LIB
python tools/ncu_summary.py gpurun_out/r2_k16tmh.ncu-rep > gpurun_out/r2_ncu_k16tmh_summary.txt 2>&1
ncu -i gpurun_out/r2_k16tmh.ncu-rep --page source --csv --print-source sass > /tmp/tmh_source.csv 2>/dev/null
python tools/sass_hist.py /tmp/tmh_source.csv --regions --stalls > gpurun_out/r2_k16tmh_sass_hist.txt 2>&1
