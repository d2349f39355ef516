mkdir -p gpurun_out
: > gpurun_out/e2e_chunks.txt
for c in 8 16 32 64; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-other-configs --no-cpu-baseline --e2e-chunks $c > /tmp/e.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/e.json')); print($c, d['value'], d['e2e']['value'])" >> gpurun_out/e2e_chunks.txt
done
python tools/h2d_bw.py >> gpurun_out/e2e_chunks.txt 2>&1
