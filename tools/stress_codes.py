"""Randomised stress of run-time code modules (jit.py) for arbitrary feed-forward codes:
random K in 3..9, B in 2..4 generators (top and bottom taps set), each code's kernels
generated and compiled at first use -- the 16x2 forms with their subset-minimum state sets
chosen per code (gen_kernels16.renorm_set) -- and decoded against the oracle on uniform,
saturated and AWGN streams with random frame length / overlap, plus a decode_batch of
random frames (decoded bits and final metrics).
usage: python tools/stress_codes.py [seed] [seconds]"""
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_13579_b200 as vt  # noqa: E402
from oracle import oracle  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
t_end = time.time() + float(sys.argv[2] if len(sys.argv) > 2 else 600)
codes = fails = runs = 0
while time.time() < t_end:
    K = int(rng.choice([3, 4, 5, 6, 7, 7, 8, 8, 9, 9]))
    B = int(rng.choice([2, 2, 3, 4]))
    gens = tuple(sorted({int(rng.integers(0, 1 << (K - 2))) << 1 | 1 | (1 << (K - 1)) for _ in range(B)}))
    if len(gens) < B:
        continue
    spec = vt.CodeSpec(K, gens)
    t0 = time.time()
    codes += 1
    for trial in range(4):
        F = int(rng.choice([7, 64, 256, 300, 1000]))
        V = int(rng.choice([0, 20, 42, 90]))
        n = int(rng.integers(2000, 60000))
        kind = trial % 3
        if kind == 0:
            q = rng.integers(-128, 128, size=(n, B)).astype(np.int8)
        elif kind == 1:
            q = (rng.choice([-128, 127], size=(n, B))).astype(np.int8)
        else:
            _, q = oracle.synthetic_stream(n, K, gens, ebn0_db=float(rng.uniform(0, 4)), seed=int(rng.integers(1 << 16)),
                                           scale=16.0)
        want = oracle.decode_stream(q, K, gens, F, V, threads=8)
        out = vt.decode_stream_device(torch.from_numpy(q).cuda(), spec, F, V)
        got = np.unpackbits(out.cpu().numpy().view(np.uint8), count=n, bitorder="little")
        runs += 1
        if not np.array_equal(got, want):
            fails += 1
            print("FAIL", K, [oct(g) for g in gens], F, V, n, kind, int((got != want).sum()), flush=True)
        if trial == 3:  # the pipelined host entry, two shards on this device (devices=[0, 0])
            hb = vt.decode_stream_host(torch.from_numpy(q).pin_memory(), spec, F, V,
                                       nchunks=int(rng.integers(1, 6)), devices=[0, 0])
            gh = np.unpackbits(hb.numpy().view(np.uint8), count=n, bitorder="little")
            runs += 1
            if not np.array_equal(gh, want):
                fails += 1
                print("FAIL host", K, [oct(g) for g in gens], F, V, n, flush=True)
    # decode_batch: frames with bits and final metrics (the final-metric kernel variants)
    nf, nl = int(rng.integers(1, 300)), int(rng.integers(1, 700))
    fr = rng.integers(-128, 128, size=(nf, B, nl)).astype(np.int8)
    mode = "hard" if rng.random() < 0.3 else "soft"
    ren = bool(rng.random() < 0.3)
    wb, wm = oracle.decode_batch(fr, K, gens, mode=mode, renormalize=ren)
    gb, gm = vt.decode_batch(fr.astype(np.float64), spec, mode=mode, renormalize=ren)
    runs += 1
    if not (np.array_equal(gb, wb) and np.array_equal(gm, wm.astype(np.float64))):
        fails += 1
        print("FAIL batch", K, [oct(g) for g in gens], nf, nl, mode, ren, flush=True)
    # decode_reference with non-uniform initial metrics (the forward/traceback kernels)
    S = 1 << (K - 1)
    init = rng.integers(-3000, 3000, size=S)
    fr1 = rng.integers(-128, 128, size=(B, int(rng.integers(1, 400)))).astype(np.int8)
    wb1, _ = oracle.decode_frame(fr1, K, gens, initial_metrics=init, renormalize=ren)
    gb1 = vt.decode_reference(fr1.astype(np.float64), spec, initial_metrics=init.astype(np.float64), renormalize=ren)
    runs += 1
    if not np.array_equal(np.asarray(gb1, dtype=np.uint8), wb1):
        fails += 1
        print("FAIL reference", K, [oct(g) for g in gens], fr1.shape, ren, flush=True)
    print(f"code K={K} {[oct(g) for g in gens]}: 4 streams + a batch ({time.time() - t0:.1f} s incl. JIT)", flush=True)
print(f"codes {codes} runs {runs} fails {fails}")
