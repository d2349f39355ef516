import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2011_13579_b200 as vt
from paper_2011_13579_b200 import fileio
from oracle import oracle
K, G = 7, (0o171, 0o133)
n, f, v = 20000, 37, 5
_, q = oracle.synthetic_stream(n, K, G, ebn0_db=2.0, seed=9, scale=16.0)
want = oracle.decode_stream(q, K, G, f, v, threads=8)
spec = vt.CodeSpec(K, G)
out = vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, f, v)
got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=n, bitorder="little")
bad = np.nonzero(got != want)[0]
print("whole stream mismatches", bad[:10], "windows", bad[:10] // f)
p = "/tmp/s.llr"
fileio.write_llr_file(q.astype(np.float64).reshape(-1), p, "half")
for per in (1, 2, 3, 1000):
    words = fileio.decode_llr_file(p, "half", spec, f, v, None, windows_per_piece=per)
    got = np.unpackbits(words.view(np.uint8), count=n, bitorder="little")
    bad = np.nonzero(got != want)[0]
    print("per", per, "mismatches", bad[:10], "windows", bad[:10] // f)
