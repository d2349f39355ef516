mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_r2.py tests/test_gpu_integration_stub.py tests/test_gpu_multitile.py -q -x > gpurun_out/pytest_r2.log 2>&1; echo "rc $?" >> gpurun_out/pytest_r2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python tools/code_bench.py k7r2 --log2n 28 --one > gpurun_out/cb.txt 2>&1
