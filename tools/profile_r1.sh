#!/bin/bash
# ncu evidence for the decoder kernel (run on the GPU box via gpurun).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:vtk_k7r2 -s 3 -c 1 -f -o gpurun_out/prof_k7r2 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof_bench.json 2>&1
ls -la gpurun_out
