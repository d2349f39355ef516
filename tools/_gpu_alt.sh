mkdir -p gpurun_out
LIB=paper_2011_13579_b200/libvitertile_b200.so
cp $LIB /tmp/lib_orig.so
cp libvariants/alt_s0.so $LIB
timeout 900 python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_parity.py tests/test_gpu_multitile.py tests/test_gpu_large.py tests/test_metric_range.py -q -x -m gpu > gpurun_out/alt_pytest.log 2>&1; echo "rc $?" >> gpurun_out/alt_pytest.log
timeout 300 python -c "
import numpy as np, torch, paper_2011_13579_b200 as vt
from oracle import oracle
for st in ('adversarial_gap_k7r2alt', 'adversarial_k7r2'):
    q = np.load('tests/golden/%s.npz' % st)['llr']
    for f, v in ((256, 42), (1000, 60), (31, 7), (24000, 0)):
        want = oracle.decode_stream(q, 7, (0o171, 0o133), f, v, threads=8)
        out = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(7, (0o171, 0o133)), f, v)
        got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=q.shape[0], bitorder='little')
        print(st, f, v, 'mismatches', int((got != want).sum()))
" >> gpurun_out/alt_pytest.log 2>&1
cp /tmp/lib_orig.so $LIB
: > gpurun_out/alt_ab.txt
SOS=$(ls libvariants/*.so | paste -sd,)
for r in 1 2; do timeout 900 python tools/code_bench.py k7r2 --log2n 28 --so $SOS >> gpurun_out/alt_ab.txt 2>&1; done
