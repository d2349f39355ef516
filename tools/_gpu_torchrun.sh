mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/tr_nccl1.json 2> gpurun_out/tr_nccl1.err; echo "rc $?" >> gpurun_out/tr_nccl1.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/tr_ref2.json 2> gpurun_out/tr_ref2.err; echo "rc $?" >> gpurun_out/tr_ref2.err
