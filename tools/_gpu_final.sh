mkdir -p gpurun_out
timeout 1500 bash tools/profile_round.sh r2 > gpurun_out/r2_profile.log 2>&1
timeout 1200 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
