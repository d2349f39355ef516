mkdir -p gpurun_out
VT_KERNEL_VARIANT=16x2tc ncu --set full --clock-control none --import-source on -k regex:vtk16tc -s 3 -c 1 -f -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_tc.ncu-rep > gpurun_out/ncu_tc_summary.txt 2>&1
ncu -i gpurun_out/prof_tc.ncu-rep --page source --csv --print-source sass > gpurun_out/tc_source.csv 2>/dev/null
python tools/sass_hist.py gpurun_out/tc_source.csv --regions --stalls > gpurun_out/tc_sass_hist.txt 2>&1
