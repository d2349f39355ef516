mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_metric_range.py tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_large.py -q -x -m gpu > gpurun_out/rset_pytest.log 2>&1; echo "rc $?" >> gpurun_out/rset_pytest.log
: > gpurun_out/rset_ab.txt
for c in k7r3 k9r2 k8r2; do
  for r in 1 2; do
    timeout 600 python tools/code_bench.py $c --log2n 28 --so libvariants/rset0.so,libvariants/rset1.so >> gpurun_out/rset_ab.txt 2>&1
  done
done
