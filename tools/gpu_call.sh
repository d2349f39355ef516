mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2>gpurun_out/bench_full.err
bash tools/profile_round.sh > gpurun_out/profile_round.log 2>&1
