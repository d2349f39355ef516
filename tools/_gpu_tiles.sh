mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tiles.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_tiles.log 2>&1; echo "rc $?" >> gpurun_out/pytest_tiles.log
python tools/tile_bench.py > gpurun_out/tile_bench.txt 2>&1
