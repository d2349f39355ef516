mkdir -p gpurun_out
cp paper_2011_13579_b200/libvitertile_b200.so /tmp/orig.so
for v in base new base new; do
  cp libvariants/$v.so paper_2011_13579_b200/libvitertile_b200.so
  timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu-baseline --no-other-configs > gpurun_out/b_$v.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'])" >> gpurun_out/ab.txt
done
cp libvariants/new.so paper_2011_13579_b200/libvitertile_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/pytest.log 2>&1; echo "rc $?" >> gpurun_out/pytest.log
cp /tmp/orig.so paper_2011_13579_b200/libvitertile_b200.so
