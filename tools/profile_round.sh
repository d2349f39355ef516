#!/bin/bash
# Round profiling evidence (run on the GPU box via gpurun): launch list of the bench
# command, one full ncu capture per decoder kernel form, the ACS-rate microbenchmark.
#   bash tools/profile_round.sh r2
R=${1:-rX}
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/${R}_launches_bench.json 2>&1
python tools/launch_summary.py gpurun_out/${R}_launches.csv "python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-other-configs" > gpurun_out/${R}_launch_list_summary.txt
ncu --set full --clock-control none --import-source on -k regex:vtk16 -s 3 -c 1 -f -o gpurun_out/${R}_k16 \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/${R}_prof_bench.json 2>&1
for c in k7r3 k9r2; do
  ncu --set full --clock-control none --import-source on -k regex:vtk16 -s 2 -c 1 -f -o gpurun_out/${R}_$c \
      python tools/code_bench.py $c --log2n 28 --one --steps 1 > /dev/null 2>&1
done
for c in k16 k7r3 k9r2; do
  python tools/ncu_summary.py gpurun_out/${R}_$c.ncu-rep > gpurun_out/${R}_ncu_${c}_summary.txt 2>&1
  ncu -i gpurun_out/${R}_$c.ncu-rep --page source --csv --print-source sass > /tmp/${c}_source.csv 2>/dev/null
  python tools/sass_hist.py /tmp/${c}_source.csv --regions --stalls > gpurun_out/${R}_${c}_sass_hist.txt 2>&1
done
rm -f gpurun_out/${R}_k7r3.ncu-rep gpurun_out/${R}_k9r2.ncu-rep
make -s -C tools/acsbench && ./tools/acsbench/acsbench > gpurun_out/${R}_acsbench.jsonl 2>&1
