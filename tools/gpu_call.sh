mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "rc $?" >> gpurun_out/pytest.log
timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/b.json 2>&1
