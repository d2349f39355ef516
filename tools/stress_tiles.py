"""Randomised stress of decode_matrix_batch (the paper's tiles on mma.sync, csrc/vt_tiles.cu)
for random feed-forward codes and configurations -- radix 2 / 4 / 4-optimised, float32 /
half accumulator, renormalisation -- against the CPU tile model (tests/tile_model.py, pinned
to the reference's own decode_matrix_batch results), and radix-2 float32 against the exact
oracle decode_batch.
usage: python tools/stress_tiles.py [seed] [seconds]"""
import os
import sys
import time

ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2011_13579_b200 as vt  # noqa: E402
import tile_model  # noqa: E402
from oracle import oracle  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
t_end = time.time() + float(sys.argv[2] if len(sys.argv) > 2 else 300)
runs = fails = 0
while time.time() < t_end:
    K = int(rng.choice([3, 4, 5, 6, 7]))
    B = int(rng.choice([2, 2, 3]))
    gens = tuple(sorted({int(rng.integers(0, 1 << (K - 2))) << 1 | 1 | (1 << (K - 1)) for _ in range(B)}))
    if len(gens) < B:
        continue
    spec = vt.CodeSpec(K, gens)
    radix = int(rng.choice([2, 4]))
    optimized = bool(radix == 4 and rng.random() < 0.5)
    half = bool(rng.random() < 0.3)
    ren = bool(rng.random() < 0.5) or half
    f, n = int(rng.integers(1, 40)), int(rng.integers(1, 300))
    llr = rng.integers(-8, 9, size=(f, B, n)).astype(np.float64) if half else \
        rng.integers(-128, 128, size=(f, B, n)).astype(np.float64)
    cfg = vt.DecoderConfig(radix=radix, optimized=optimized, renormalize=ren,
                           policy=vt.PrecisionPolicy(accumulator="half" if half else "single"))
    try:
        res = vt.decode_matrix_batch(llr, spec, cfg)
    except ValueError as exc:  # configurations the reference rejects too (e.g. no dragonfly groups)
        print("rejected", K, [oct(g) for g in gens], radix, optimized, half, str(exc)[:60])
        continue
    wb, wm, _ = tile_model.decode(llr.astype(np.float32), spec, radix, optimized, half, ren)
    runs += 1
    ok = np.array_equal(res.bits, wb) and np.array_equal(res.final_metric, wm, equal_nan=True)
    if radix == 2 and not half:
        ob, om = oracle.decode_batch(llr.astype(np.int64), K, gens, renormalize=ren)
        # (decode_batch reports the renormalised final metric, decode_matrix_batch max + offsets)
        ok = ok and np.array_equal(res.bits, ob) and (ren or np.array_equal(res.final_metric, om.astype(np.float64)))
    if not ok:
        fails += 1
        print("FAIL", K, [oct(g) for g in gens], radix, optimized, half, ren, f, n, flush=True)
print(f"runs {runs} fails {fails}")
