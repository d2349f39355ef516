"""Soft-decision BER curves of the three BASELINE codes on the GPU (K=7 r1/2,
K=7 r1/3, K=9 r1/2), each through its default kernel form, with the Eb/N0 at
BER 1e-3 and 1e-5.  Coding-gain sanity check: the stronger codes must reach a
given BER at a lower Eb/N0.  Writes profiles/<tag>_ber_codes.json.
usage: python tools/ber_codes.py [tag] [bits_per_point]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13579_b200 as vt  # noqa: E402
from paper_2011_13579_b200 import channel as ch  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
bits = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
codes = {"K=7 r1/2 (171,133)": (7, (0o171, 0o133)), "K=7 r1/3 (133,171,165)": (7, (0o133, 0o171, 0o165)),
         "K=9 r1/2 (753,561)": (9, (0o753, 0o561))}
grid = [round(0.5 + 0.25 * i, 2) for i in range(19)]
out = {"bits_per_point": bits, "llr": "int8, q = clamp(rint(16 y), -127, 127); frames of 1024 bits; GPU Philox channel",
       "codes": {}}
for name, (k, gens) in codes.items():
    spec = vt.CodeSpec(k, gens)
    t0 = time.time()
    pts = ch.ber_sweep(spec, grid, bits, seed=51, mode="soft")
    dt = time.time() - t0
    valid = [p for p in pts if p.valid]
    res = {"seconds": round(dt, 2), "points": [p.__dict__ for p in pts]}
    for target in (1e-3, 1e-5):
        try:
            res[f"ebn0_at_{target:g}"] = round(ch.ebn0_at_ber(valid, target), 3)
        except Exception as exc:  # target not bracketed by the grid
            res[f"ebn0_at_{target:g}"] = None
            res[f"note_{target:g}"] = str(exc)
    out["codes"][name] = res
    print(name, {k_: v for k_, v in res.items() if k_ != "points"}, flush=True)
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(f"profiles/{tag}_ber_codes.json", "w"), indent=1)
