mkdir -p gpurun_out
for r in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --no-other-configs --no-cpu-baseline > gpurun_out/b20_$r.json 2>gpurun_out/b20_$r.err; done
timeout 600 python tools/code_bench.py k7r2 --log2n 28 --steps 20 > gpurun_out/b20_cb.txt 2>&1
