mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/exp1.txt
python tools/code_bench.py k7r2 --log2n 28 --one >> gpurun_out/exp1.txt 2>&1
VT_CTAS_PER_SM=1 python tools/code_bench.py k7r2 --log2n 28 --one >> gpurun_out/exp1.txt 2>&1
VT_CTAS_PER_SM=1 python tools/code_bench.py k7r2 --log2n 28 --one --frame 1024 >> gpurun_out/exp1.txt 2>&1
python tools/code_bench.py k7r2 --log2n 28 --one --frame 1024 >> gpurun_out/exp1.txt 2>&1
VT_CTAS_PER_SM=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:vtk16 -c 2 python tools/code_bench.py k7r2 --log2n 28 --one --steps 1 >> gpurun_out/exp1.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:vtk16 -c 2 python tools/code_bench.py k7r2 --log2n 28 --one --steps 1 >> gpurun_out/exp1.txt 2>&1
