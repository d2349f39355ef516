mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/f3_pytest_all.log 2>&1; echo "rc $?" >> gpurun_out/f3_pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "rc $?" >> gpurun_out/f3_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f3_bench.json 2>gpurun_out/f3_bench.err
