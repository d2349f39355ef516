"""Randomised stress of the API entry points around the kernels: decode_batch
(soft / hard / renormalize; bits and final metrics vs the oracle on sampled
frames), window-range pieces (fileio.decode_llr_file) and the pipelined host
entry (random chunk counts) vs the device-resident decode.
usage: python tools/stress_api.py [seed] [seconds]"""
import os, sys, time, tempfile
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np, torch
import paper_2011_13579_b200 as vt
from paper_2011_13579_b200 import fileio
from oracle import oracle
CODES = [(7, (0o171, 0o133)), (7, (0o133, 0o171, 0o165)), (9, (0o753, 0o561)), (8, (0o247, 0o371)), (5, (0o23, 0o35))]
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
t_end = time.time() + float(sys.argv[2] if len(sys.argv) > 2 else 300)
runs = fails = 0
tmp = tempfile.mkdtemp()
while time.time() < t_end:
    k, gens = CODES[rng.integers(len(CODES))]
    spec = vt.CodeSpec(k, gens)
    b = len(gens)
    what = rng.integers(3)
    ok = True
    if what == 0:  # decode_batch
        f, n = int(rng.integers(1, 30000)), int(rng.integers(1, 700))
        if f * n > 40_000_000:
            continue
        llrs = rng.integers(-128, 128, size=(f, b, n)).astype(np.float64)
        mode = "hard" if rng.random() < 0.2 else "soft"
        ren = bool(rng.random() < 0.3)
        bits, metric = vt.decode_batch(llrs, spec, mode=mode, renormalize=ren)
        sel = np.unique(rng.integers(0, f, size=min(f, 40)))
        src = llrs[sel]
        if mode == "hard":
            src = np.where(src >= 0, 1, -1)
        wb, wm = oracle.decode_batch(src.astype(np.int8), k, gens)
        ok = np.array_equal(bits[sel], wb) and (ren or np.array_equal(metric[sel], wm.astype(np.float64)))
        desc = f"batch f={f} n={n} mode={mode} ren={ren}"
    else:
        F = int(rng.choice([32, 100, 256, 1000]))
        V = int(rng.choice([0, 21, 42, 150]))
        n = int(rng.integers(1, 60000)) * F // 4 + int(rng.integers(0, F))
        n = max(n, 1)
        q = rng.integers(-128, 128, size=(n, b)).astype(np.int8)
        whole = vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, F, V).cpu()
        if what == 1:
            p = os.path.join(tmp, "q.llr")
            fileio.write_llr_file(q.astype(np.float32).reshape(-1), p, "single")
            per = int(rng.integers(1, 5000))
            got = torch.from_numpy(fileio.decode_llr_file(p, "single", spec, F, V, windows_per_piece=per))
            desc = f"pieces F={F} V={V} n={n} per={per}"
        else:
            ch = int(rng.integers(1, 20))
            got = vt.decode_stream_host(torch.from_numpy(q).pin_memory(), spec, F, V, nchunks=ch)
            desc = f"host F={F} V={V} n={n} chunks={ch}"
        ok = torch.equal(got, whole)
    runs += 1
    if not ok:
        fails += 1
        print("FAIL", k, oct(gens[0]), desc, flush=True)
print("runs", runs, "fails", fails)
