"""ctypes front end of the C oracle (viterbi_oracle.c) plus numpy restatements
of the reference's synthetic-data helpers.  TEST INFRASTRUCTURE ONLY.

Parity pinning: every function here is checked against golden vectors that
the reference itself produced (tests/golden/make_golden.py, tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

__all__ = [
    "VtoCode",
    "load",
    "build",
    "decode_frame",
    "decode_batch",
    "decode_stream",
    "encode_batch",
    "generate_bits",
    "modulate_awgn",
    "quantize",
    "synthetic_stream",
    "plan_windows",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


class VtoCode(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("B", ctypes.c_int), ("gens", ctypes.c_uint32 * 8)]


def build() -> str:
    """Compile the C oracle with make (gcc); returns the library path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.POINTER
        lib.vto_decode_frame.argtypes = [p(VtoCode), p(ctypes.c_int64), ctypes.c_int64, p(ctypes.c_int64),
                                         ctypes.c_int, p(ctypes.c_uint8), p(ctypes.c_int64)]
        lib.vto_decode_batch.argtypes = [p(VtoCode), p(ctypes.c_int64), ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_int, p(ctypes.c_uint8), p(ctypes.c_int64)]
        lib.vto_decode_stream.argtypes = [p(VtoCode), p(ctypes.c_int8), ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, p(ctypes.c_uint8), ctypes.c_int]
        lib.vto_decode_stream_range.argtypes = [p(VtoCode), p(ctypes.c_int8), ctypes.c_int64, ctypes.c_int64,
                                                ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                                p(ctypes.c_uint8), ctypes.c_int]
        lib.vto_encode_batch.argtypes = [p(VtoCode), p(ctypes.c_uint8), ctypes.c_int64, ctypes.c_int64,
                                         p(ctypes.c_uint8)]
        for fn in ("vto_decode_frame", "vto_decode_batch", "vto_decode_stream",
                   "vto_decode_stream_range", "vto_encode_batch"):
            getattr(lib, fn).restype = ctypes.c_int
        _lib = lib
    return _lib


def _code(constraint_length: int, generators) -> VtoCode:
    c = VtoCode()
    c.K = int(constraint_length)
    c.B = len(generators)
    for i, g in enumerate(generators):
        c.gens[i] = int(g)
    return c


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def decode_frame(llr, constraint_length: int, generators, initial_metrics=None, renormalize=False):
    """reference.py:181-191 decode_reference (soft) on an integer (B, N) frame.
    Returns (bits uint8 (N,), final metric int)."""
    llr = np.ascontiguousarray(np.asarray(llr), dtype=np.int64)
    b, n = llr.shape
    bits = np.empty(n, dtype=np.uint8)
    fm = np.zeros(1, dtype=np.int64)
    init = None if initial_metrics is None else np.ascontiguousarray(initial_metrics, dtype=np.int64)
    rc = load().vto_decode_frame(ctypes.byref(_code(constraint_length, generators)), _ptr(llr, ctypes.c_int64),
                                 n, None if init is None else _ptr(init, ctypes.c_int64), int(renormalize),
                                 _ptr(bits, ctypes.c_uint8), _ptr(fm, ctypes.c_int64))
    if rc:
        raise RuntimeError(f"oracle vto_decode_frame failed ({rc})")
    return bits, int(fm[0])


def decode_batch(llrs, constraint_length: int, generators, mode="soft", renormalize=False):
    """reference.py:194-206 decode_batch on integer (F, B, N) frames.
    Returns (bits uint8 (F, N), final metrics int64 (F,))."""
    llrs = np.asarray(llrs)
    if mode == "hard":
        llrs = np.where(llrs >= 0, 1, -1)
    llrs = np.ascontiguousarray(llrs, dtype=np.int64)
    f, b, n = llrs.shape
    bits = np.empty((f, n), dtype=np.uint8)
    fm = np.empty(f, dtype=np.int64)
    rc = load().vto_decode_batch(ctypes.byref(_code(constraint_length, generators)), _ptr(llrs, ctypes.c_int64),
                                 f, n, int(renormalize), _ptr(bits, ctypes.c_uint8), _ptr(fm, ctypes.c_int64))
    if rc:
        raise RuntimeError(f"oracle vto_decode_batch failed ({rc})")
    return bits, fm


def decode_stream(llr_nb, constraint_length: int, generators, frame_len: int, overlap: int,
                  threads: int = 1, windows=None):
    """framing.py:96-141 decode_stream with the reference decoder, on an int8
    stage-major (N, B) stream.  Returns uint8 bits (N,).  ``windows`` =
    (w_begin, w_end) restricts decoding to a window range (other bits stay 0)."""
    llr_nb = np.ascontiguousarray(llr_nb, dtype=np.int8)
    n = llr_nb.shape[0]
    out = np.zeros(n, dtype=np.uint8)
    code = _code(constraint_length, generators)
    if windows is None:
        rc = load().vto_decode_stream(ctypes.byref(code), _ptr(llr_nb, ctypes.c_int8), n, int(frame_len),
                                      int(overlap), _ptr(out, ctypes.c_uint8), int(threads))
    else:
        rc = load().vto_decode_stream_range(ctypes.byref(code), _ptr(llr_nb, ctypes.c_int8), n, int(frame_len),
                                            int(overlap), int(windows[0]), int(windows[1]),
                                            _ptr(out, ctypes.c_uint8), int(threads))
    if rc:
        raise RuntimeError(f"oracle vto_decode_stream failed ({rc})")
    return out


def encode_batch(bits2d, constraint_length: int, generators) -> np.ndarray:
    """codes.py:216-230 encode_batch: (F, N) bits -> (F, N, B) coded bits."""
    bits2d = np.ascontiguousarray(bits2d, dtype=np.uint8)
    f, n = bits2d.shape
    out = np.empty((f, n, len(generators)), dtype=np.uint8)
    rc = load().vto_encode_batch(ctypes.byref(_code(constraint_length, generators)), _ptr(bits2d, ctypes.c_uint8),
                                 f, n, _ptr(out, ctypes.c_uint8))
    if rc:
        raise RuntimeError("oracle vto_encode_batch failed")
    return out


def _rng(seed: int, *stream: int) -> np.random.Generator:
    # channel.py:34-35: Philox keyed by SeedSequence((seed, *stream))
    return np.random.Generator(np.random.Philox(np.random.SeedSequence((int(seed), *map(int, stream)))))


def generate_bits(n: int, seed: int, stream: int = 0) -> np.ndarray:
    """channel.py:69-73 generate_bits."""
    return _rng(seed, stream, 0).integers(0, 2, size=n, dtype=np.uint8)


def sigma_standard(ebn0_db: float, rate: float) -> float:
    """channel.py:52-57 ChannelModel.sigma, 'standard' convention."""
    return math.sqrt(1.0 / (2.0 * rate * 10.0 ** (ebn0_db / 10.0)))


def modulate_awgn(coded_bits, ebn0_db: float, rate: float, seed: int, stream: int = 0) -> np.ndarray:
    """channel.py:76-87 modulate_awgn (standard sigma convention)."""
    bits = np.asarray(coded_bits)
    sigma = sigma_standard(ebn0_db, rate)
    noise = _rng(seed, stream, 1).normal(0.0, 1.0, size=bits.shape) * sigma
    return 1.0 - 2.0 * bits.astype(np.float64) + noise


def quantize(y, scale: float = 16.0) -> np.ndarray:
    """SURVEY.md §8(d) quantiser: q = clamp(rint(scale * y), -127, 127) as int8."""
    return np.clip(np.rint(np.asarray(y, dtype=np.float64) * scale), -127, 127).astype(np.int8)


def synthetic_stream(n: int, constraint_length: int, generators, ebn0_db: float = 3.0, seed: int = 0,
                     scale: float = 16.0):
    """Bits + int8 stage-major (N, B) LLR stream of an AWGN/BPSK channel
    (SURVEY.md §8(d) synthetic recipe)."""
    bits = generate_bits(n, seed, 0)
    coded = encode_batch(bits[None, :], constraint_length, generators)[0]  # (N, B)
    y = modulate_awgn(coded, ebn0_db, 1.0 / len(generators), seed, 0)
    return bits, quantize(y, scale)


def plan_windows(n: int, frame_len: int, overlap: int):
    """framing.py:68-83 plan_frames in closed form: list of (start, stop, emit_start, emit_stop)."""
    out = []
    for e0 in range(0, n, frame_len):
        e1 = min(e0 + frame_len, n)
        out.append((max(0, e0 - overlap), min(n, e1 + overlap), e0, e1))
    return out
