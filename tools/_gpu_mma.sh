mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_metric_range.py -q -x -m gpu -k "mma" > gpurun_out/mma_pytest.log 2>&1; echo "rc $?" >> gpurun_out/mma_pytest.log
: > gpurun_out/mma_ab.txt
for r in 1 2; do timeout 600 python tools/code_bench.py k7r2 --log2n 28 --variants 16x2,16x2mma,16x2tc >> gpurun_out/mma_ab.txt 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vtk16mma -s 2 -c 1 -f -o gpurun_out/r2_k16mma python tools/code_bench.py k7r2 --log2n 28 --variants 16x2mma --steps 1 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/r2_k16mma.ncu-rep > gpurun_out/r2_ncu_k16mma_summary.txt 2>&1
ncu -i gpurun_out/r2_k16mma.ncu-rep --page source --csv --print-source sass > /tmp/mma_source.csv 2>/dev/null
python tools/sass_hist.py /tmp/mma_source.csv --regions --stalls > gpurun_out/r2_k16mma_sass_hist.txt 2>&1
