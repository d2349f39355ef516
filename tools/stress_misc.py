"""Randomised stress of the remaining reference-API paths: forward_batch /
traceback_batch consistency with decode_batch (random codes, renormalisation,
initial metrics), and exact pairing of channel.run_point(rng="numpy") with the
oracle for every code and decision mode.
usage: python tools/stress_misc.py [seed] [seconds]"""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_2011_13579_b200 as vt
from paper_2011_13579_b200 import channel as ch, reference as R
from oracle import oracle
CODES = [(3, (0o7, 0o5)), (5, (0o23, 0o35)), (7, (0o171, 0o133)), (7, (0o133, 0o171, 0o165)), (8, (0o247, 0o371)),
         (9, (0o753, 0o561))]
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
t_end = time.time() + float(sys.argv[2] if len(sys.argv) > 2 else 300)
runs = fails = 0
while time.time() < t_end:
    k, gens = CODES[rng.integers(len(CODES))]
    spec = vt.CodeSpec(k, gens)
    b = len(gens)
    if rng.random() < 0.5:
        f, n = int(rng.integers(1, 200)), int(rng.integers(1, 300))
        llrs = rng.integers(-128, 128, size=(f, b, n)).astype(np.float64)
        surv, lam, hist = R.forward_batch(llrs, spec, keep_history=bool(rng.random() < 0.3))
        bits = R.traceback_batch(surv, lam, spec)
        db, dm = vt.decode_batch(llrs, spec)
        ok = np.array_equal(bits, db) and np.array_equal(lam.max(axis=1), dm)
        if hist is not None:
            ok = ok and np.array_equal(hist[:, -1, :], lam)
        desc = f"forward f={f} n={n}"
    else:
        mode = "hard" if rng.random() < 0.3 else "soft"
        fl = int(rng.choice([64, 100, 1024]))
        ebn0 = float(rng.uniform(0, 4))
        seed, pi = int(rng.integers(1000)), int(rng.integers(50))
        p = ch.run_point(spec, ebn0, 20_000, seed=seed, frame_len=fl, point_index=pi, rng="numpy", mode=mode)
        frames = -(-20_000 // fl)
        data = ch.generate_bits(frames * fl, seed, pi).reshape(frames, fl)
        y = ch.modulate_awgn(vt.encode_batch(data, spec), ch.ChannelModel(ebn0, seed=seed), 1.0 / b, pi)
        q = np.where(y >= 0, 1, -1) if mode == "hard" else np.clip(np.rint(y * 16), -127, 127)
        wb, _ = oracle.decode_batch(np.transpose(q.astype(np.int8), (0, 2, 1)), k, gens)
        desc = f"ber {mode} fl={fl}"
        ok = p.n == frames * fl and p.errors == int(np.count_nonzero(wb != data))
    runs += 1
    if not ok:
        fails += 1
        print("FAIL", k, oct(gens[0]), desc, flush=True)
print("runs", runs, "fails", fails)
