# A/B of library variants over codes: CODES="k7r3 k9r2" SOS="libvariants/a.so,..." OUT=name
mkdir -p gpurun_out
: > gpurun_out/$OUT.txt
for c in $CODES; do
  for r in 1 2; do
    timeout 900 python tools/code_bench.py $c --log2n 28 --so $SOS >> gpurun_out/$OUT.txt 2>&1
  done
done
