#!/bin/bash
# Round profiling evidence (run on the GPU box via gpurun): launch list of the bench
# command, one full ncu capture of the decoder kernel, the ACS-rate microbenchmark.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/launches_bench.json 2>&1
python tools/launch_summary.py gpurun_out/launches.csv "python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs" > gpurun_out/launch_list_summary.txt
ncu --set full --clock-control none --import-source on -k regex:vtk16 -s 3 -c 1 -f -o gpurun_out/prof_k16 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/prof_bench.json 2>&1
python tools/ncu_summary.py gpurun_out/prof_k16.ncu-rep > gpurun_out/ncu_k16_summary.txt 2>&1
ncu -i gpurun_out/prof_k16.ncu-rep --page source --csv --print-source sass > gpurun_out/k16_source.csv 2>/dev/null
python tools/sass_hist.py gpurun_out/k16_source.csv --regions --stalls > gpurun_out/k16_sass_hist.txt 2>&1
make -s -C tools/acsbench && ./tools/acsbench/acsbench > gpurun_out/acsbench.jsonl 2>&1
