#!/bin/bash
mkdir -p gpurun_out
VT_KERNEL_VARIANT=16x2 ncu --set full --clock-control none --import-source on -k regex:vtk16_k7r2 -s 3 -c 1 -f -o gpurun_out/prof_k16 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/prof16_bench.json 2>&1
python tools/ncu_summary.py gpurun_out/prof_k16.ncu-rep
