mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r2h_pytest.log 2>&1; echo "rc $?" >> gpurun_out/r2h_pytest.log
for c in k7r2 k7r3 k9r2; do timeout 300 python tools/code_bench.py $c --log2n 28 --one >> gpurun_out/r2h.txt 2>&1; done
