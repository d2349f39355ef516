"""Run the 16x2tc kernel on several stream sizes in subprocesses with timeouts."""
import os, subprocess, sys
CODE = r'''
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2011_13579_b200 as vt
from oracle import oracle
n, f, v = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
_, q = oracle.synthetic_stream(n, 7, (0o171, 0o133), ebn0_db=2.0, seed=3, scale=16.0)
out = vt.decode_stream_device(torch.from_numpy(q).cuda(), vt.CodeSpec(7, (0o171, 0o133)), f, v)
torch.cuda.synchronize()
got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=n, bitorder="little")
want = oracle.decode_stream(q, 7, (0o171, 0o133), f, v, threads=8)
print("mismatches", int(np.count_nonzero(got != want)))
'''
for n, f, v in [(1 << 18, 256, 42), (1 << 16, 256, 42), (65536 + 256 * 3, 256, 42), (4096, 256, 42), (60000, 256, 42)]:
    env = dict(os.environ)
    try:
        r = subprocess.run([sys.executable, "-c", CODE, str(n), str(f), str(v)], env=env, capture_output=True,
                           text=True, timeout=40)
        print(n, f, v, "rc", r.returncode, r.stdout.strip()[-200:], r.stderr.strip()[-300:], flush=True)
    except subprocess.TimeoutExpired:
        print(n, f, v, "TIMEOUT", flush=True)
