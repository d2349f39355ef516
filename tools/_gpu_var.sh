# A/B of library variants: timing (code_bench) + ncu DRAM/L2 metrics of one steady-state launch
mkdir -p gpurun_out
OUT=gpurun_out/var_${TAG:-x}.txt
: > $OUT
LIB=paper_2011_13579_b200/libvitertile_b200.so
cp $LIB /tmp/lib_orig.so
CODE=${CODE:-k7r2}
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum"
for v in $VARS; do
  cp libvariants/$v.so $LIB
  for r in 1 2; do echo -n "[$v] " >> $OUT; timeout 300 python tools/code_bench.py $CODE --log2n 28 --one >> $OUT 2>&1; done
  [ -n "$NONCU" ] && continue
  echo "[$v] ncu" >> $OUT
  timeout 300 ncu --metrics $M --clock-control none -k regex:vtk16 -s 2 -c 1 python tools/code_bench.py $CODE --log2n 28 --one --steps 1 2>&1 | grep -E "dram__|gpu__time|lts__|inst_issued|inst_executed" >> $OUT
done
cp /tmp/lib_orig.so $LIB
