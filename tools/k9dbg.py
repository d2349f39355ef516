import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle, paper_2011_13579_b200 as vt
spec = vt.CodeSpec(9, (0o753, 0o561))
n = 4096
_, q = oracle.synthetic_stream(n, 9, (0o753, 0o561), 3.0, 1)
w = vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, 256, 42)
torch.cuda.synchronize()
got = np.unpackbits(w.cpu().numpy().view(np.uint8), count=n, bitorder='little')
want = oracle.decode_stream(q, 9, (0o753, 0o561), 256, 42)
print('mismatch', np.count_nonzero(got != want))
