"""Golden files for the on-disk formats, written BY THE REFERENCE's own writers.

Run in the build container (where /root/reference exists):
    python tests/golden/make_fileio_golden.py
Imports the unmodified reference CLI module (pkg/src/vitertile/cli.py:31-62) and
writes small bit/LLR files plus the arrays they encode into tests/golden/fileio/.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from vitertile.cli import write_bit_file, write_llr_file  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fileio")
os.makedirs(OUT, exist_ok=True)
rng = np.random.default_rng(2011_13579)
arrays = {}
for n in (0, 1, 13, 32, 33, 64, 1000):
    bits = rng.integers(0, 2, n).astype(np.uint8)
    arrays[f"bits_{n}"] = bits
    write_bit_file(bits, os.path.join(OUT, f"bits_{n}.bin"))
llr = rng.integers(-128, 128, 2 * 300).astype(np.float64)
arrays["llr_int"] = llr
write_llr_file(llr, os.path.join(OUT, "llr_int_half.bin"), "half")
write_llr_file(llr, os.path.join(OUT, "llr_int_single.bin"), "single")
llr_f = rng.normal(0, 20, 2 * 50)
arrays["llr_float"] = llr_f
write_llr_file(llr_f, os.path.join(OUT, "llr_float_half.bin"), "half")
write_llr_file(llr_f, os.path.join(OUT, "llr_float_single.bin"), "single")
np.savez(os.path.join(OUT, "arrays.npz"), **arrays)
print("wrote", sorted(os.listdir(OUT)))
