"""md5 of the decoded bits of a fixed synthetic stream (A/B correctness of library variants):
python tools/bits_hash.py k7r2 [log2n] -- run once per swapped-in library and compare."""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13579_b200 as vt  # noqa: E402
from bench import make_stream  # noqa: E402
from tools.code_bench import CODES  # noqa: E402

code = sys.argv[1]
log2n = int(sys.argv[2]) if len(sys.argv) > 2 else 26
k, gens = CODES[code]
dev = torch.device("cuda", 0)
n = 1 << log2n
for f, v in ((256, 42), (100, 7), (1024, 0)):
    _, q = make_stream(torch, n + 1234, seed=5, device=dev, gens=gens, k=k)
    o = torch.zeros((n + 1234 + 31) // 32, dtype=torch.int32, device=dev)
    vt.decode_stream_device(q, vt.CodeSpec(k, gens), f, v, out=o)
    torch.cuda.synchronize()
    print(code, f, v, hashlib.md5(o.cpu().numpy().tobytes()).hexdigest(), flush=True)
