"""Round-2 golden vectors, generated FROM THE REFERENCE ITSELF (build container only):
    python tests/golden/make_golden_r2.py
Imports the unmodified reference from /root/reference/pkg/src and records into
tests/golden/golden_r2.npz:

* ``codes``: decode_stream / decode_batch on int8 streams for codes that are NOT
  built into the library (generated at run time by paper_2011_13579_b200/jit.py):
  K=7 (133,171) (the headline code with its generators swapped), a non-standard
  K=5 (25,33), a B=4 code K=5 (25,33,37,31), K=9 rate 1/3 (557,663,711), K=4 (13,17).
* ``dragonfly``: compute_bomat / identical_bomat_classes / find_dragonfly_groups
  (rho = 1, 2) for every conftest/BASELINE code incl. K=8/9, where the radix-4
  optimisation is not effective (codes.py:351-412).
* ``ber``: run_point's own sample recipe (generate_bits / encode_batch /
  modulate_awgn, channel.py:113-136) quantised to int8 (q = clamp(rint(16 y)))
  and decoded by the reference's decode_batch: error counts per Eb/N0 point (and
  per frame: errors come in bursts, so confidence intervals use the frame-level
  variance), plus the reference's float-LLR run_point count on the same samples.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from vitertile.channel import ChannelModel, generate_bits, modulate_awgn, run_point  # noqa: E402
from vitertile.codes import (CodeSpec, compute_bomat, encode_batch, find_dragonfly_groups,  # noqa: E402
                             identical_bomat_classes)
from vitertile.framing import decode_stream, plan_frames  # noqa: E402
from vitertile.matrix import DecoderConfig, decode_matrix_batch, pack_radix4  # noqa: E402
from vitertile.tile import PrecisionPolicy  # noqa: E402
from vitertile.reference import decode_batch  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_r2.npz")

JIT_CODES = {
    "k7r2s": (7, ("133", "171")),
    "k5x": (5, ("25", "33")),
    "k5r4": (5, ("25", "33", "37", "31")),
    "k9r3": (9, ("557", "663", "711")),
    "k4x": (4, ("13", "17")),
}
STD_CODES = {
    "k7r2": (7, ("171", "133")), "k7r3": (7, ("133", "171", "165")), "k9r2": (9, ("753", "561")),
    "k9r2t": (9, ("561", "753")), "k3r2": (3, ("7", "5")), "k4r2": (4, ("17", "15")),
    "k5r2": (5, ("23", "35")), "k6r2": (6, ("53", "75")), "k8r2": (8, ("247", "371")),
}
BER_POINTS = [1.0, 2.0, 3.0, 4.0]
BER_BITS = 1 << 20
BER_SEED = 11


def spec_of(k, polys):
    return CodeSpec.from_octal(k, polys)


def awgn_q(spec, n, ebn0, seed, scale=16.0):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2, n, dtype=np.uint8)
    coded = encode_batch(bits[None, :], spec)[0]
    sigma = ChannelModel(ebn0).sigma(1.0 / spec.outputs_per_bit)
    y = 1.0 - 2.0 * coded + rng.normal(0.0, sigma, coded.shape)
    return np.clip(np.rint(scale * y), -127, 127).astype(np.int8)


def main():
    data, index = {}, {"codes": {**JIT_CODES, **STD_CODES}, "cases": []}
    rng = np.random.default_rng(2011_13579 + 2)

    def add(kind, **kw):
        key = f"{kind}_{len(index['cases']):03d}"
        index["cases"].append({"key": key, "kind": kind, **{k: v for k, v in kw.items() if not isinstance(v, np.ndarray)}})
        for k, v in kw.items():
            if isinstance(v, np.ndarray):
                data[f"{key}_{k}"] = v
        return key

    # --- codes the library is not built with
    for name, (k, polys) in JIT_CODES.items():
        spec = spec_of(k, polys)
        b = spec.outputs_per_bit
        for tag, q, f, v in (
                ("awgn2", awgn_q(spec, 3000, 2.0, k * 7 + b), 256, 42),
                ("uniform_partial_tail", rng.integers(-128, 128, size=(2345, b)).astype(np.int8), 200, 30),
                ("ties", rng.integers(-1, 2, size=(1500, b)).astype(np.int8), 64, 9),
                ("v0", awgn_q(spec, 700, 1.0, k + 3), 100, 0)):
            bits = decode_stream(q.T.astype(np.float64), spec, plan_frames(q.shape[0], f, v), decoder="reference")
            add("stream", code=name, tag=tag, n=int(q.shape[0]), frame_len=f, overlap=v, llr=q,
                bits=np.packbits(bits, bitorder="little"))
        frames = rng.integers(-128, 128, size=(5, b, 77)).astype(np.float64)
        bits, metric = decode_batch(frames, spec)
        add("batch", code=name, llr=frames.astype(np.int8), bits=bits, metric=metric)

    # --- the tile decoder with the half accumulator (tile.py:87-89) and long frames whose
    #     binary16 metrics overflow to inf, plus single precision on codes not in golden.npz
    for name, (k, polys) in {**STD_CODES, "k7r2s": JIT_CODES["k7r2s"], "k5x": JIT_CODES["k5x"]}.items():
        spec = spec_of(k, polys)
        b = spec.outputs_per_bit
        for n, scale in ((41, 127), (200, 40), (700, 127)):
            frames = np.clip(np.rint(rng.normal(0, scale / 2, size=(3, b, n))), -128, 127)
            for radix in (2, 4):
                if radix == 4 and 2 * b > 4:
                    continue
                for opt in ((False, True) if radix == 4 else (False,)):
                    for acc in ("half", "single"):
                        for renorm in (False, True):
                            if acc == "single" and (n != 200 or not renorm):
                                continue
                            cfg = DecoderConfig(radix=radix, optimized=opt, renormalize=renorm,
                                                policy=PrecisionPolicy(accumulator=acc))
                            with np.errstate(all="ignore"):
                                res = decode_matrix_batch(frames, spec, cfg)
                            add("tile", code=name, n=n, radix=radix, optimized=opt, accumulator=acc,
                                renormalize=renorm, llr=frames.astype(np.int8), bits=res.bits,
                                metric=np.asarray(res.final_metric, dtype=np.float64),
                                counter=np.array([res.counter.mma_ops, res.counter.survivor_write_passes,
                                                  res.counter.stages]))

    # --- dragonfly structures (radix-2 and radix-4)
    for name, (k, polys) in STD_CODES.items():
        spec = spec_of(k, polys)
        for rho in (1, 2):
            if rho * spec.outputs_per_bit > 8:
                continue
            nd = spec.num_dragonflies(rho)
            bomats = np.stack([compute_bomat(f, rho, spec) for f in range(nd)])
            classes = [list(c) for c in identical_bomat_classes(rho, spec)]
            groups = [{"representative": g.representative, "members": list(g.members),
                       "permutations": {str(f): list(p) for f, p in g.permutations.items()}}
                      for g in find_dragonfly_groups(rho, spec)]
            eff = bool(pack_radix4(spec, True).optimization_effective) if rho == 2 and 2 * spec.outputs_per_bit <= 4 \
                else None
            add("dragonfly", code=name, rho=rho, classes=classes, groups=groups, bomats=bomats, r4_effective=eff)

    # --- BER points: the reference's own samples, int8-quantised, reference decoder
    spec = spec_of(7, ("171", "133"))
    flen = 1024
    frames = BER_BITS // flen
    for idx, ebn0 in enumerate(BER_POINTS):
        ch = ChannelModel(ebn0, "standard", BER_SEED)
        bits = generate_bits(frames * flen, BER_SEED, idx).reshape(frames, flen)
        y = modulate_awgn(encode_batch(bits, spec), ch, 0.5, idx)  # (F, N, B)
        q = np.clip(np.rint(16.0 * y), -127, 127)
        dec, _ = decode_batch(np.transpose(q, (0, 2, 1)), spec)
        frame_errors = np.count_nonzero(dec != bits, axis=1).astype(np.int32)
        errors_q = int(frame_errors.sum())
        ref_float = run_point(spec, ebn0, BER_BITS, seed=BER_SEED, frame_len=flen, point_index=idx)
        add("ber", code="k7r2", ebn0_db=ebn0, point_index=idx, seed=BER_SEED, frame_len=flen, n=int(bits.size),
            errors_int8=errors_q, errors_float=int(ref_float.errors), frame_errors=frame_errors)
        print(f"BER point {ebn0} dB: int8 {errors_q} errors, float {ref_float.errors} / {bits.size}")

    data["index_json"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **data)
    print("wrote", OUT, len(index["cases"]), "cases")


if __name__ == "__main__":
    main()
