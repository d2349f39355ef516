"""BER curves on the GPU (soft and hard decision, K=7 r1/2) next to the
reference's published anchors (pkg/test_output.txt:19-23).  Writes
profiles/<tag>_ber.json and .csv."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2011_13579_b200 as vt  # noqa: E402
from paper_2011_13579_b200 import channel as ch  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
bits = int(float(sys.argv[2])) if len(sys.argv) > 2 else 100_000_000
spec = vt.default_spec()
grid = [round(1.0 + 0.25 * i, 2) for i in range(25)]
t0 = time.time()
soft = ch.ber_sweep(spec, grid, bits, seed=50, mode="soft")
hard = ch.ber_sweep(spec, grid, bits, seed=50, mode="hard")
dt = time.time() - t0
sx = ch.ebn0_at_ber([p for p in soft if p.valid], 1e-3)
hx = ch.ebn0_at_ber([p for p in hard if p.valid], 1e-3)
out = {
    "bits_per_point": bits, "points": len(grid) * 2, "seconds": round(dt, 2),
    "info_bits_per_s": round(len(grid) * 2 * bits / dt),
    "soft_ebn0_at_1e-3": round(sx, 3), "hard_ebn0_at_1e-3": round(hx, 3), "gap_db": round(hx - sx, 3),
    "reference_anchor": {"soft": 2.77, "hard": 4.92, "gap": 2.15,
                         "source": "pkg/test_output.txt:19 (reference decoder, float LLRs, 1e6 bits/point)"},
    "llr": "int8, q = clamp(rint(16 y), -127, 127); frames of 1024 bits from the zero state; GPU Philox channel",
    "soft": [p.__dict__ for p in soft], "hard": [p.__dict__ for p in hard],
}
os.makedirs("profiles", exist_ok=True)
json.dump(out, open(f"profiles/{tag}_ber.json", "w"), indent=1)
ch.write_ber_csv(soft, f"profiles/{tag}_ber_soft.csv")
ch.write_ber_csv(hard, f"profiles/{tag}_ber_hard.csv")
print(json.dumps({k: v for k, v in out.items() if k not in ("soft", "hard")}))
