"""Generate golden vectors for the vitertile hot path FROM THE REFERENCE ITSELF.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It imports the unmodified reference package from /root/reference/pkg/src and
records inputs + outputs of decode_stream / decode_batch / decode_matrix_batch /
encode_batch / generate_bits / modulate_awgn into tests/golden/golden.npz.
The GPU box never needs the reference: tests read only the .npz.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from vitertile.channel import ChannelModel, generate_bits, modulate_awgn  # noqa: E402
from vitertile.codes import CodeSpec, encode_batch  # noqa: E402
from vitertile.framing import decode_stream, plan_frames  # noqa: E402
from vitertile.matrix import DecoderConfig, decode_matrix_batch  # noqa: E402
from vitertile.reference import decode_batch  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

CODES = {
    "k7r2": (7, ("171", "133")),
    "k7r3": (7, ("133", "171", "165")),
    "k9r2": (9, ("753", "561")),
    "k9r2t": (9, ("561", "753")),
    "k3r2": (3, ("7", "5")),
    "k4r2": (4, ("17", "15")),
    "k5r2": (5, ("23", "35")),
    "k6r2": (6, ("53", "75")),
    "k8r2": (8, ("247", "371")),
}


def spec_of(name):
    k, polys = CODES[name]
    return CodeSpec.from_octal(k, polys)


def awgn_stream(spec, n, ebn0, seed, scale=16.0):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, n, dtype=np.uint8)
    coded = encode_batch(bits[None, :], spec)[0]  # (N, B)
    sigma = ChannelModel(ebn0).sigma(1.0 / spec.outputs_per_bit)
    y = 1.0 - 2.0 * coded + rng.normal(0.0, sigma, coded.shape)
    return np.clip(np.rint(scale * y), -127, 127).astype(np.int8)  # (N, B)


def main():
    data = {}
    index = []
    rng = np.random.default_rng(2011_13579)

    def add_stream(tag, code, q, f, v):
        spec = spec_of(code)
        plan = plan_frames(q.shape[0], f, v)
        bits = decode_stream(q.T.astype(np.float64), spec, plan, decoder="reference")
        key = f"stream_{len(index):03d}"
        data[key + "_llr"] = q
        data[key + "_bits"] = np.packbits(bits, bitorder="little")
        index.append({"key": key, "kind": "stream", "tag": tag, "code": code, "n": int(q.shape[0]),
                      "frame_len": int(f), "overlap": int(v)})

    for code in ("k7r2", "k7r3", "k9r2"):
        b = spec_of(code).outputs_per_bit
        add_stream("awgn3", code, awgn_stream(spec_of(code), 4096, 3.0, 1), 256, 42)
        add_stream("awgn1_partial_tail", code, awgn_stream(spec_of(code), 5000, 1.0, 2), 256, 42)
        add_stream("uniform_int8", code, rng.integers(-128, 128, size=(3000, b)).astype(np.int8), 256, 42)
        add_stream("all_zero_ties", code, np.zeros((600, b), dtype=np.int8), 256, 42)
        add_stream("saturated", code,
                   (127 * (2 * rng.integers(0, 2, size=(1200, b)) - 1)).astype(np.int8), 100, 20)
        add_stream("small_levels", code, rng.integers(-2, 3, size=(2000, b)).astype(np.int8), 64, 20)
        add_stream("f100_v0", code, awgn_stream(spec_of(code), 777, 2.0, 3), 100, 0)
        add_stream("single_window", code, awgn_stream(spec_of(code), 50, 2.0, 4), 256, 42)
        add_stream("one_stage", code, awgn_stream(spec_of(code), 1, 2.0, 5), 256, 42)
        add_stream("f1_v3", code, awgn_stream(spec_of(code), 40, 2.0, 6), 1, 3)
        add_stream("f33_v7", code, awgn_stream(spec_of(code), 500, 2.0, 7), 33, 7)
        add_stream("f512_v64", code, awgn_stream(spec_of(code), 3000, 2.5, 8), 512, 64)
    for code in ("k9r2t", "k3r2", "k4r2", "k5r2", "k6r2", "k8r2"):
        add_stream("awgn2", code, awgn_stream(spec_of(code), 2000, 2.0, 9), 256, 42)
        add_stream("uniform_int8", code,
                   rng.integers(-128, 128, size=(900, spec_of(code).outputs_per_bit)).astype(np.int8), 128, 30)

    # decode_batch (reference.py:194-206): frames (F, B, N) with integer LLRs
    for code in ("k7r2", "k7r3", "k9r2", "k3r2", "k8r2"):
        spec = spec_of(code)
        for n in (1, 2, 7, 64, 300):
            llrs = rng.integers(-128, 128, size=(8, spec.outputs_per_bit, n)).astype(np.int8)
            for mode in ("soft", "hard"):
                for renorm in (False, True):
                    if renorm and mode == "hard":
                        continue
                    bits, metric = decode_batch(llrs.astype(np.float64), spec, mode=mode, renormalize=renorm)
                    key = f"batch_{len(index):03d}"
                    data[key + "_llr"] = llrs
                    data[key + "_bits"] = bits
                    data[key + "_metric"] = metric
                    index.append({"key": key, "kind": "batch", "code": code, "n": n, "mode": mode,
                                  "renormalize": renorm})

    # decode_matrix_batch (matrix.py:342-386) on int LLRs: bits, metric, counters
    for code in ("k7r2", "k5r2"):
        spec = spec_of(code)
        for n in (1, 11, 64, 201):
            llrs = rng.integers(-128, 128, size=(6, spec.outputs_per_bit, n)).astype(np.int8)
            for radix, opt in ((2, False), (4, False), (4, True)):
                for renorm in (False, True):
                    res = decode_matrix_batch(llrs.astype(np.float64), spec,
                                              DecoderConfig(radix=radix, optimized=opt, renormalize=renorm))
                    key = f"matrix_{len(index):03d}"
                    data[key + "_llr"] = llrs
                    data[key + "_bits"] = res.bits
                    data[key + "_metric"] = np.asarray(res.final_metric, dtype=np.float64)
                    data[key + "_counter"] = np.array([res.counter.mma_ops, res.counter.survivor_write_passes,
                                                       res.counter.stages], dtype=np.int64)
                    index.append({"key": key, "kind": "matrix", "code": code, "n": n, "radix": radix,
                                  "optimized": opt, "renormalize": renorm})

    # encode_batch (codes.py:216-230)
    for code in ("k7r2", "k7r3", "k9r2", "k3r2"):
        bits = rng.integers(0, 2, size=(3, 257), dtype=np.uint8)
        key = f"encode_{len(index):03d}"
        data[key + "_in"] = bits
        data[key + "_out"] = encode_batch(bits, spec_of(code))
        index.append({"key": key, "kind": "encode", "code": code})

    # channel sources (channel.py:69-87)
    key = f"channel_{len(index):03d}"
    data[key + "_bits"] = generate_bits(1000, seed=5, stream=2)
    coded = rng.integers(0, 2, size=(4, 50, 2), dtype=np.uint8)
    data[key + "_coded"] = coded
    data[key + "_y"] = modulate_awgn(coded, ChannelModel(3.0, seed=11), 0.5, stream=4)
    index.append({"key": key, "kind": "channel", "seed": 5, "stream": 2, "ebn0": 3.0, "mod_seed": 11,
                  "mod_stream": 4, "rate": 0.5})

    data["index_json"] = np.frombuffer(json.dumps({"codes": CODES, "cases": index}).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **data)
    print(f"wrote {OUT}: {len(index)} cases, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
