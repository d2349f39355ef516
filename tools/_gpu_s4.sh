mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s4_pytest_all.log 2>&1; echo "rc $?" >> gpurun_out/s4_pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4_smoke.log 2>&1; echo "rc $?" >> gpurun_out/s4_smoke.log
timeout 900 python bench.py > gpurun_out/s4_bench.json 2>gpurun_out/s4_bench.err
timeout 1800 bash tools/profile_round.sh r2b > gpurun_out/s4_profile_round.log 2>&1
