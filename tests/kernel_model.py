"""Bit-level numpy model of the generated sm_100a kernel algorithm (test-only).

It mirrors vt_common.cuh + gen_kernels.py step by step -- end-aligned BL-stage
chunks with zero-LLR front padding, int32 metrics M = lambda<<16 | history,
+2^p on the i1 candidate, renormalisation folded into the first stage of a
chunk, BL-bit history blocks, traceback j_prev = h & (S-1),
bits = ((h | j<<BL) >> (K-1)) & (2^BL-1) -- so the design can be checked
against the oracle on the CPU, independently of the CUDA code.
"""
from __future__ import annotations

import numpy as np


def _pattern_tables(K, gens):
    k = K - 1
    S = 1 << k
    H = S // 2
    j = np.arange(S)
    i0 = 2 * (j & (H - 1))
    i1 = i0 + 1
    u = j >> (k - 1)

    def pat(i):
        reg = (u << k) | i
        return sum(((np.vectorize(lambda x: bin(x).count("1") & 1)(g & reg)) << b) for b, g in enumerate(gens))

    return S, i0, i1, pat(i0), pat(i1)


def decode_stream_model(llr_nb: np.ndarray, K: int, gens, F: int, V: int, BL: int | None = None) -> np.ndarray:
    """BL = history block length (the generated kernels use 16)."""
    if BL is None:
        BL = 16
    n, B = llr_nb.shape
    S, i0, i1, p0, p1 = _pattern_tables(K, gens)
    nw = -(-n // F)
    lmax = min(n, F + 2 * V)
    nc = -(-lmax // BL)
    head = min(n, F + V)
    b_lo = max(0, (BL * nc - head) // BL)
    out = np.zeros(n, dtype=np.uint8)
    signs = np.array([[1 - 2 * ((p >> b) & 1) for b in range(B)] for p in range(1 << B)], dtype=np.int64)
    for w in range(nw):
        e0 = w * F
        e1 = min(e0 + F, n)
        s = max(0, e0 - V)
        stop = min(n, e1 + V)
        g0 = stop - BL * nc
        M = np.zeros(S, dtype=np.int64)
        rfold = 0
        fields = {}
        for c in range(nc):
            for q in range(BL):
                st = g0 + BL * c + q
                ll = llr_nb[st].astype(np.int64) if st >= s else np.zeros(B, dtype=np.int64)
                L = ll << 16
                D = signs @ L - (rfold if q == 0 else 0)
                E = D + (1 << q)
                c1 = M[i1] + E[p1]
                c0 = M[i0] + D[p0]
                M = np.maximum(c0, c1)
                assert np.all(np.abs(M) < 2 ** 31), "int32 overflow"
            if c >= b_lo:
                fields[c] = (M & 0xFFFF).copy()
            M = M & ~np.int64(0xFFFF)
            rfold = int(M[0])
        key = M | (S - 1 - np.arange(S))
        jst = S - 1 - (int(key.max()) & 0xFFFF)
        for b in range(nc - 1, -1, -1):
            gb = g0 + BL * b
            h = int(fields[b][jst]) if b in fields else 0
            bits = ((h | (jst << BL)) >> (K - 1)) & ((1 << BL) - 1)
            jst = ((jst << BL) | h) & (S - 1)
            for i in range(BL):
                pos = gb + i
                if e0 <= pos < e1:
                    out[pos] = (bits >> i) & 1
            if gb <= e0:
                break
    return out
