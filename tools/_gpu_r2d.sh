mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/d_gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/d_pytest.log 2>&1; echo "rc $?" >> gpurun_out/d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/d_smoke.log 2>&1; echo "rc $?" >> gpurun_out/d_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/d_bench.json 2>gpurun_out/d_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/d_ref.json 2>gpurun_out/d_ref.err
