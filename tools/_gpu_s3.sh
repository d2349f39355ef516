mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s3_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s3_pytest_all.log 2>&1; echo "rc $?" >> gpurun_out/s3_pytest_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo "rc $?" >> gpurun_out/s3_smoke.log
timeout 900 python bench.py > gpurun_out/s3_bench.json 2>gpurun_out/s3_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/s3_bench_torchrun.json 2>gpurun_out/s3_bench_torchrun.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s3_bench_ref.json 2>gpurun_out/s3_bench_ref.err
