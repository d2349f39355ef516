"""Bit-level model of the generated 16x2 kernels' arithmetic (test-only).

Mirrors gen_kernels16.py / gen_kernels16m.py for ONE 16-bit half (the two
windows of a register never interact): per state U = Lambda * 2^L + h; every
LLR term enters biased (U_b = (l+128) << L, N_b = (256 << L) - U_b); the i1
candidate carries +2^q at group stage q (stored groups only); the cheap middle
stage stores metric - S(p0) and the next stage absorbs the offsets; group ends
mask, store and clear the L-bit fields and renormalise the next group by
Lambda_0 - S_b, by the exact minimum or by the minimum over a small state set
(renorm_set; the generator's own choice); traceback
j_prev = ((j << L) | h) & (S-1).  Every value the kernels compute in a 16-bit
half is asserted to stay in [0, 2^16) -- the range argument of the generators,
exercised on the CPU against the oracle and the adversarial streams.
"""
from __future__ import annotations

import os
import sys

import numpy as np

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "paper_2011_13579_b200", "csrc"))

LIM = 1 << 16


def _par(x: int) -> int:
    return bin(x).count("1") & 1


def _gen(K: int, gens):
    if K in (8, 9):
        from gen_kernels16m import Gen16M
        return Gen16M("model", K, tuple(gens), {8: 2, 9: 4}[K])
    from gen_kernels16 import Gen16
    return Gen16("model", K, tuple(gens))


def _in_range(x, what):
    assert np.all(x >= 0) and np.all(x < LIM), f"{what} leaves the 16-bit half"


def decode_stream_model16(llr_nb: np.ndarray, K: int, gens, F: int, V: int) -> np.ndarray:
    g = _gen(K, gens)
    L, CH, Sb, cheap, xmin = g.L, g.CH, g.Sb, g.cheap, g.xmin
    multilane = hasattr(g, "rsets")
    # alternating form (VT_ALT16, no-final-metric kernel): body stages C A C A C A, the
    # renormalisation folded into absorbing stages 3 and 5 from references after stages 1, 3
    alt = bool(getattr(g, "alt", False))
    if alt:
        Sb = g.Sb_alt
        alt_T = np.array(g.alt_T)
    # renormalisation reference per group position in the body: all states (exact minimum),
    # the subset T (gen_kernels16.renorm_set) or state 0
    if multilane and g.rsets:
        refsets = [np.array(r[0]) for r in g.rsets]
    elif not multilane and getattr(g, "rset", None):
        refsets = [np.array(g.rset)] * g.GPB
    else:
        refsets = None
    n, B = llr_nb.shape
    k = K - 1
    S = 1 << k
    full = (1 << B) - 1
    j = np.arange(S)
    u = j >> (k - 1)
    i0 = (j << 1) & (S - 1)
    i1 = i0 | 1

    def pat(i, uu):
        reg = (uu << k) | i
        return sum(np.array([_par(int(g_ & r)) for r in reg]) << b for b, g_ in enumerate(gens))

    p0, p1 = pat(i0, u), pat(i1, u)
    c0 = pat((i0 << 1) & (S - 1), i0 >> (k - 1))  # class of i0 at the previous (cheap) stage
    c1 = pat((i1 << 1) & (S - 1), i1 >> (k - 1))

    lmax = min(n, F + 2 * V)
    nc = -(-lmax // CH)
    ng = nc * (CH // L)
    head = min(n, F + V)
    b_lo = max(0, (CH * nc - head) // L)
    out = np.zeros(n, dtype=np.uint8)
    for w in range(-(-n // F)):
        e0, e1 = w * F, min(w * F + F, n)
        s, stop = max(0, e0 - V), min(n, e1 + V)
        g0 = stop - CH * nc
        m = np.full(S, (Sb << L) if (cheap or multilane) else 0, dtype=np.int64)
        r_alt = {}
        negR = 0  # renormalisation R = Lambda_ref*2^L - Sb*2^L, subtracted in group stage 0
        fields = {}
        s_prev = None
        for gi in range(ng):
            flag = 1 if gi >= b_lo else 0
            for gq in range(L):
                st = g0 + gi * L + gq
                ll = llr_nb[st].astype(np.int64) if st >= s else np.zeros(B, dtype=np.int64)
                U = (ll + 128) << L
                N = (256 << L) - U
                Sp = np.array([sum(int(N[b] if (p >> b) & 1 else U[b]) for b in range(B)) for p in range(1 << B)])
                qb = (gi % g.GPB) * L + gq  # body position
                if alt and qb % 2 == 0:
                    T = Sp[p0 ^ full] - Sp[p0] + flag * (1 << gq)
                    cand1 = m[i1] + T
                    _in_range(cand1, "cheap candidate")
                    m = np.maximum(cand1, m[i0])
                    s_prev = Sp
                elif alt:
                    r = r_alt.get(qb, 0) if qb in (3, 5) else 0
                    d = s_prev[c0] + Sp[p0] - r
                    e = s_prev[c1] + Sp[p1] + flag * (1 << gq) - r
                    cand0, cand1 = m[i0] + d, m[i1] + e
                    _in_range(cand0, "candidate 0")
                    _in_range(cand1, "candidate 1")
                    m = np.maximum(cand0, cand1)
                    if qb in (1, 3):  # reference for the absorbing stage two stages on
                        lm_ = LIM - (1 << L)
                        r_alt[qb + 2] = (int(m[alt_T].min()) & lm_) - (Sb << L)
                elif cheap and gq == 1:
                    T = Sp[p0 ^ full] - Sp[p0] + 2 * flag  # i1 candidate relative to i0's offset
                    cand1 = m[i1] + T
                    _in_range(cand1, "cheap candidate")
                    m = np.maximum(cand1, m[i0])
                    s_prev = Sp
                elif cheap and gq == 2:
                    d = s_prev[c0] + Sp[p0]
                    e = s_prev[c1] + Sp[p1] + flag * (1 << gq)
                    cand0, cand1 = m[i0] + d, m[i1] + e
                    _in_range(cand0, "candidate 0")
                    _in_range(cand1, "candidate 1")
                    m = np.maximum(cand0, cand1)
                else:
                    r = negR if gq == 0 else 0
                    cand0 = m[i0] + Sp[p0] - r
                    cand1 = m[i1] + Sp[p1] - r + flag * (1 << gq)
                    _in_range(cand0, "candidate 0")
                    _in_range(cand1, "candidate 1")
                    m = np.maximum(cand0, cand1)
            # group end: renormalisation reference, fields, clear
            lm = LIM - (1 << L)
            if alt:
                pass
            elif refsets is not None:
                ref = int(m[refsets[gi % g.GPB]].min()) & lm
                # the subset minimum is within 256 * W_T = Sb of the exact minimum
                assert int(m.min()) & lm >= ref - (Sb << L)
            else:
                ref = (int(m.min()) if xmin else int(m[0])) & lm
            if not alt:
                negR = ref - (Sb << L)
            h = m & ((1 << L) - 1)
            if gi >= b_lo:
                fields[gi] = h.copy()
            m = m - h
        jst = int(np.argmax(m))  # lowest index on ties (reference.py:138)
        for gi in range(ng - 1, -1, -1):
            gs = g0 + gi * L
            hh = int(fields[gi][jst]) if gi in fields else 0
            bits = jst >> (k - L)
            for i in range(L):
                pos = gs + i
                if e0 <= pos < e1:
                    out[pos] = (bits >> i) & 1  # the newest input is the state's top bit
            jst = ((jst << L) | hh) & (S - 1)
            if gs <= e0:
                break
    return out
