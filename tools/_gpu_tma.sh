mkdir -p gpurun_out
./tools/tma_probe > gpurun_out/tma_probe.txt 2>&1
for i in 1 2; do
python tools/code_bench.py k7r2 --log2n 28 --one >> gpurun_out/tma_cb.txt 2>&1
VT_NO_TMA=1 python tools/code_bench.py k7r2 --log2n 28 --one >> gpurun_out/tma_cb.txt 2>&1
done
python tools/code_bench.py k7r3 --log2n 28 --one >> gpurun_out/tma_cb.txt 2>&1
VT_NO_TMA=1 python tools/code_bench.py k7r3 --log2n 28 --one >> gpurun_out/tma_cb.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_r2.py tests/test_gpu_integration_stub.py tests/test_gpu_fuzz.py -q -x > gpurun_out/pytest_tma.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tma.log
