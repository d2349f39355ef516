"""Host-side cost of one small decode call (launch-bound regime): wall time per
vt.decode_stream_device call on a 256-stage stream, and per raw C-ABI call."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13579_b200 as vt  # noqa: E402

spec = vt.CodeSpec(7, (0o171, 0o133))
q = torch.randint(-128, 128, (256, 2), dtype=torch.int8, device="cuda")
out = torch.zeros(8, dtype=torch.int32, device="cuda")
for _ in range(50):
    vt.decode_stream_device(q, spec, 256, 42, out=out)
torch.cuda.synchronize()
for n in (1000,):
    t0 = time.perf_counter()
    for _ in range(n):
        vt.decode_stream_device(q, spec, 256, 42, out=out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"decode_stream_device 256 stages: {1e6 * (t1 - t0) / n:.1f} us/call host, {1e6 * (t2 - t0) / n:.1f} us/call incl. sync")
