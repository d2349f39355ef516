#!/bin/bash
# Sustained-vs-burst decode rate with power/clock samples (nvidia-smi, 50 ms):
#   bash tools/power_probe.sh [code]   -> gpurun_out/power_probe.txt
CODE=${1:-k7r2}
OUT=gpurun_out/power_probe.txt; mkdir -p gpurun_out; : > $OUT
nvidia-smi --query-gpu=power.limit,power.default_limit,power.max_limit,clocks.max.sm,temperature.gpu --format=csv >> $OUT
for steps in 20 200 2000; do
  nvidia-smi --query-gpu=timestamp,power.draw,clocks.sm,temperature.gpu,clocks_event_reasons.active --format=csv,noheader -lms 50 > /tmp/smi_$steps.csv &
  P=$!
  python tools/code_bench.py $CODE --log2n 28 --one --steps $steps >> $OUT 2>&1
  kill $P; sleep 0.5
  echo "steps=$steps samples:" >> $OUT
  python - "$steps" >> $OUT <<'PY'
import sys, statistics
rows=[l.strip().split(', ') for l in open(f"/tmp/smi_{sys.argv[1]}.csv") if l.strip()]
pw=[float(r[1].split()[0]) for r in rows if r[1][0].isdigit()]
ck=[float(r[2].split()[0]) for r in rows if r[2][0].isdigit()]
busy=[(p,c,r[4]) for p,c,r in zip(pw,ck,rows) if p>300]
if busy:
    print(f"  n={len(busy)} power median {statistics.median(p for p,_,_ in busy):.0f} W max {max(p for p,_,_ in busy):.0f} W; sm clock median {statistics.median(c for _,c,_ in busy):.0f} min {min(c for _,c,_ in busy):.0f} MHz; reasons {sorted(set(r for _,_,r in busy))}")
else:
    print("  no busy samples", len(rows))
PY
done
