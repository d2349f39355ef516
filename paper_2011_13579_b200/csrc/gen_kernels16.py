#!/usr/bin/env python3
"""Generator for the packed 16x2 ACS kernels (two windows per thread), K = 7
(K = 8, 9: gen_kernels16m.py, the same forms over 2 / 4 lanes).

Each 32-bit register m_j holds the metric of state j for TWO windows: window
A in the low 16 bits, window B in the high 16 bits.  Both windows walk the
same trellis, so one carry-free `IMAD` (candidate i1, FMA pipe) + one
`VIADDMNMX.U16x2` (fused add of candidate i0 + unsigned max, ALU pipe) advance
state j of both windows: half the issue slots per state update of the s32
kernels (gen_kernels.py).  `tools/pipe_bench.cu` measures the VIADD.16x2 +
VIADDMNMX.U16x2 pair at 101 state updates/cycle/SM (the roofline peak);
the cheap middle stage (stage()) needs only the VIADDMNMX.

Per 16-bit half:  U = Lambda * 2^L + h  (unsigned), where
  * h (L bits) records the survivor decisions of the current L-stage history
    group (candidate i1 carries +2^q at group stage q, so unsigned max applies
    the reference tie rule take1 = cand1 >= cand0, reference.py:121);
  * Lambda is the biased path metric: every LLR term enters as l+128 or 128-l
    (both >= 0), so each stage adds delta + 128*B >= 0; at each group start the
    metrics are renormalised by Lambda_0 - S_b (S_b bounds the metric spread),
    keeping Lambda in [0, 2*S_b + L*256*B] < 2^(16-L) (L = 3 for K=7 r1/2); K=7
    r1/3 renormalises by a per-half minimum instead (Gen16.xmin: over a small
    state set T, renorm_set, within 256 * W_T of the exact minimum), which
    shrinks the span and also fits L = 3.  Per-half arithmetic is modular; the
    true values stay in range, so the unsigned max is exact.
At each group end the L-bit fields are masked out, packed 4 states per word
(12 bits per half), streamed to the scratch slot and cleared.  The traceback
walks groups: j_prev = ((j << L) | h) & (S-1), decoded bits =
(j >> (K-1-L)) & (2^L - 1) (vt_common.cuh TracebackLite<K, L>), fed by a
shared-memory ring of whole history groups prefetched 4 groups ahead.
"""
from __future__ import annotations

import os

from gen_kernels import parity

NT = int(os.environ.get("VT_NT16", "128"))  # threads per CTA of the 16x2 kernels (2 windows each)
# (the traceback's ring addressing is (j & 48) << log2(NT) = (j >> 4) * NT * 16; it was hard-coded for
# 128 threads until round 2d, which is why VT_NT16=64 faulted in round 2b.  Measured in round 2d:
# 64 -> 165.9, 256 -> 162.5 vs 167.3 Gbps, bits identical)
assert NT in (64, 128, 256), "the 16x2 kernels are generated for 64-, 128- or 256-thread CTAs"
NTS = NT.bit_length() - 1
# VT_LOCK16 (with VT_NT16=256): a barrier after every LLR chunk keeps the two warps of each SM
# sub-partition (warps w and w + 4) at the same point of the 22.6 KB loop body, so one warp's
# instruction-cache fills serve the other (no L0 reuse otherwise).  1: a named
# barrier per warp pair, 2: the whole CTA
LOCK = int(os.environ.get("VT_LOCK16", "0"))

CH_BODIES = 2  # loop bodies per LLR chunk
MINB16 = 1  # CTAs per SM bound (3 forces a 168-register cap: spills, measured 16% slower with the ring traceback)


# Emission seeds picked by measurement (tools/_gpu_var.sh / _gpu_ab2.sh over VT_SEED16 / VT_SEED16M =
# 0..7, 2^28 stages, profiles/r2_schedule_sweep.txt, r2_seed_ab.txt).  Re-swept after the subset
# minimum (round 2b): K=7 r1/3 seed 0 143.65 (seeds 1-7: 141.9-143.5), K=9 seed 5 36.90 (35.9-36.8);
# K=7 r1/2 keeps the default order (the fastest of 13).
MEASURED_SEEDS = {(9, (0o753, 0o561)): 5}


def history_bits(K: int, B: int) -> int:
    dmax = 128 * B
    sb = 2 * (K - 1) * dmax
    for L in (6, 3, 2, 1):
        if (K - 1) % L == 0 and 2 * sb + L * 2 * dmax < (1 << (16 - L)):
            return L
    raise ValueError("no history width fits")


def weight_table(K: int, gens: tuple[int, ...]) -> list[int]:
    """w[e] = Hamming weight of the encoder output of the K-1 input bits e from the zero
    state (newest bit at the register MSB as codes.py:183-193).  Two paths from one
    state that end in states s and s' (s' = s ^ e: the end state is the last K-1 inputs)
    differ in at most w[e] output bits, so |Lambda(s) - Lambda(s')| <= 256 * w[e] for
    |l| <= 128 -- at every stage, also inside the window's first K-1 stages (all initial
    metrics are equal) and over zero-LLR padding."""
    k = K - 1
    out = []
    for e in range(1 << k):
        reg, w = 0, 0
        for t in range(k):
            reg = (reg >> 1) | (((e >> t) & 1) << k)
            w += sum(parity(g & reg) for g in gens)
        out.append(w)
    return out


def spread_weight(K: int, gens: tuple[int, ...]) -> int:
    """Max Hamming weight of the output difference of two K-1-stage paths from the same
    state (= encoder output weight of a nonzero input sequence from the zero state,
    newest bit at the register MSB as codes.py:183-193): the metric spread is at most
    256 * this for |l| <= 128."""
    return max(weight_table(K, gens))


_RSET_CACHE: dict = {}


def renorm_set(K: int, gens: tuple[int, ...], wmax: int, allowed=None, max_size: int = 6,
               budget: int = 300000):
    """Smallest state set T (|T| <= max_size, members from `allowed`) whose minimum metric
    is within 256 * W_T of the exact minimum, W_T = max_m min_{t in T} w[t ^ m] <= wmax
    (weight_table's bound applied to the minimising state m and its nearest member of T).
    Renormalising by R = min_T Lambda - 256 * W_T then keeps every metric in
    [0, 256 * W_T + Delta] at a group start, like the exact minimum up to 256 * W_T, for
    |T| - 1 min operations instead of a tree over all states.  Set cover by depth-first
    search (branch on the lowest uncovered state).  Returns (sorted T, W_T) or None."""
    key = (K, tuple(gens), wmax, None if allowed is None else tuple(sorted(allowed)), max_size)
    if key in _RSET_CACHE:
        return _RSET_CACHE[key]
    S = 1 << (K - 1)
    w = weight_table(K, gens)
    full = (1 << S) - 1
    pool = set(range(S)) if allowed is None else set(allowed)
    ball = [e for e in range(S) if w[e] <= wmax]
    cover = {t: sum(1 << (t ^ e) for e in ball) for t in pool}
    nodes = [0]

    def dfs(cov: int, n: int, T: list):
        nodes[0] += 1
        if cov == full:
            return T
        if n == 0 or nodes[0] > budget:
            return None
        free = ~cov & full
        m = (free & -free).bit_length() - 1
        for e in ball:
            t = m ^ e
            if t in cover:
                r = dfs(cov | cover[t], n - 1, T + [t])
                if r is not None:
                    return r
        return None

    res = None
    for n in range(1, max_size + 1):
        nodes[0] = 0
        r = dfs(0, n, [])
        if r is not None:
            T = sorted(r)
            res = (T, max(min(w[t ^ m] for t in T) for m in range(S)))
            break
    _RSET_CACHE[key] = res
    return res


class Gen16:
    def __init__(self, name: str, K: int, gens: tuple[int, ...], tc: bool = False, mma: bool = False):
        self.name = name
        self.K = K
        self.k = K - 1
        self.S = 1 << self.k
        assert self.S >= 16, "16x2 kernels pack 16 states per uint4 of history words"
        self.gens = gens
        self.B = len(gens)
        self.dmax = 128 * self.B
        delta = 256 * spread_weight(K, gens)
        # Exact-minimum renormalisation (xmin): when renormalising by state 0 forces
        # history groups narrower than 3 bits (K=7 r1/3), renormalise by the exact
        # per-half minimum over the 2^(K-1) states instead (~S/2 VIMNMX3.U16x2 per
        # group): the metrics then span [Sb', Sb' + Delta] at a group start instead of
        # [Sb - Delta, Sb + Delta], which fits 3-bit groups.
        L = history_bits(K, self.B)
        self.xmin = False
        if L < 3 and self.k % 3 == 0 and delta + 3 * 2 * self.dmax < (1 << 13):
            L, self.xmin = 3, True
        self.L = L
        self.P = self.k  # body length: the state->register naming returns to the identity
        self.GPB = self.P // self.L  # history groups per body
        # per-body LLR realignment from the staged rows (4-body chunks: half the per-chunk
        # bookkeeping per group, 3 LLR words per window in registers instead of 6)
        # even groups per body: the traceback ring alternates statically (odd counts, i.e.
        # 2-bit groups, are left to the s32 kernels: generate() checks `supported`)
        self.supported = self.GPB % 2 == 0
        self.pbr = not tc
        self.tma = self.pbr and os.environ.get("VT_TMA16", "1") == "1"  # TMA LLR staging (interior warps)
        # 5-body (30-stage) chunks: the traceback settles once per chunk, and 5 bodies x 6 bits
        # + < 32 unwritten bits fit its 64-bit accumulator (6 bodies measured +0.6% but need a
        # mid-chunk settle, -2.5%)
        self.CHB = int(os.environ.get("VT_CHB16", "5")) if self.pbr else CH_BODIES
        self.CH = self.P * self.CHB  # LLR chunk (stages)
        self.GPB = self.P // self.L  # history groups per body
        self.Sb = 2 * self.k * self.dmax
        # Cheap middle stage (see stage()): needs 3-bit groups, an even number of groups
        # per body and complementary branch patterns of the two predecessors (every
        # generator taps the oldest register bit), and a renormalisation target
        # Sb' >= Delta + 2*dmax with Sb' + Delta + L*2*dmax < 2^(16-L), where Delta =
        # 256 * W is the metric-spread bound from the code's maximum output-difference
        # weight W over K-1 stages (|l| <= 128 per LLR).
        comp = all(self.pattern(((j << 1) & (self.S - 1)) | 1, j >> (self.k - 1)) ==
                   self.pattern((j << 1) & (self.S - 1), j >> (self.k - 1)) ^ ((1 << self.B) - 1)
                   for j in range(self.S))
        sbc = delta + 2 * self.dmax
        # (not with xmin: for B = 3 the offset stage needs 64 + 64 combo adds per group,
        # measured slower than the plain stage: 120.0 vs 123.6 Gbps for K=7 r1/3)
        self.cheap = (not self.xmin and self.L == 3 and self.supported and comp and
                      sbc + delta + self.L * 2 * self.dmax < (1 << (16 - self.L)))
        # Subset minimum (round 2): renormalise by the minimum over a small state set T
        # (renorm_set) instead of the exact minimum over all 2^(K-1) states: the metrics
        # then span [0, Sb' + Delta] with Sb' = 256 * W_T at a group start, which must still
        # leave L stages of growth below 2^(16-L).  K=7 r1/3: |T| = 6, W_T = 7 (7936 < 8192):
        # 3 VIMNMX instead of a 32-instruction tree per group.  VT_RSET=0: the exact minimum.
        self.clri = int(os.environ.get("VT_CLRI16", "0"))  # xmin group end: IMAD clears (see group_end)
        self.gebf = os.environ.get("VT_GEBF16", "0") == "1"
        self.rset = None
        if self.xmin and os.environ.get("VT_RSET", "1") == "1":
            wmax = ((1 << (16 - L)) - 1 - delta - L * 2 * self.dmax) // 256
            r = renorm_set(K, gens, wmax) if wmax >= 0 else None
            if r is not None:
                self.rset = r[0]
                self.Sb_rset = 256 * r[1]
        if self.xmin:  # the minimum renormalises to 0 (the subset minimum to Sb' = 256 * W_T)
            self.Sb = self.Sb_rset if self.rset else 0
            assert self.Sb + delta + L * 2 * self.dmax < (1 << (16 - L)), "metric range"
        elif self.cheap:
            self.Sb = sbc
        self.NWC = -(-self.CH * self.B // 4)
        self.NL = -(-(self.NWC * 4 + 15) // 16)
        while self.NWC + 4 > 4 * self.NL:
            self.NL += 1
        self.NWB = -(-self.P * self.B // 4)  # LLR words per body (per-body realignment)
        if self.pbr:  # a body's words start anywhere in the row: 15 + CH*B bytes + one word of lookahead
            self.NL = -(-(15 + self.CH * self.B + 4) // 16)
        self.lines: list[str] = []
        # L2 policy of the history stores: the oldest quarter of the stored groups (lowest gs,
        # longest lifetime) evict-first, the rest evict-last.  The live history set (~1 tile
        # slot per CTA, 242 MB at config 2) exceeds L2 whatever the split; the
        # split measured -5% DRAM bytes and +1% speed (167.3 vs 165.6 Gbps, 2 runs each).
        # VT_SEED16: semantically neutral emission choices (butterfly order of the full
        # stages, traceback step before/after the history store).  ptxas's schedule -- the
        # issue efficiency, 67-72% -- depends on them: seeds 1-8 measured 161.1-167.4 Gbps,
        # the default order (0) 167.4
        self.seed = int(os.environ.get("VT_SEED16", str(MEASURED_SEEDS.get((K, tuple(gens)), 0))))
        import random
        self.rng = random.Random(self.seed)
        # last-tile traceback 8 groups deep through the freed LLR rows (needs TBD = 4 and rows
        # of >= 4 ring entries).  Measured (2^24 / 2^26 / 2^28 stages): r1/3 +2.5% / - / +0.1%;
        # r1/2 +2.4% / -1.0% / -0.6% (ptxas reallocates the body's registers), so r1/3 only
        self.DRAIN8 = (self.pbr and os.environ.get("VT_DRAIN8", "0" if self.cheap_candidate() else "1") == "1"
                       and 4 * ((-(-(15 + self.P * int(os.environ.get("VT_CHB16", "5")) * self.B + 4) // 16)) | 1)
                       >= 4 * (self.S // 16) and "VT_TBD16" not in os.environ)
        self.EF = int(os.environ.get("VT_EF16", "64" if self.cheap_candidate() else "0"))  # 1/256 of the stored groups
        self.efc = os.environ.get("VT_EFC16", "0") == "1"  # evict-first split per chunk instead of per group
        # TMEM history window (see tmh_* below): 16 of a tile's stored-group positions live in the
        # CTA's tensor memory (256 columns x 128 lanes: one 16-word group per thread and column
        # block) instead of the HBM scratch slot
        self.tmh = (os.environ.get("VT_TMH16", "0") == "1" and not tc and not mma and self.pbr and NT == 128
                    and self.S == 64)
        self.TMW = 16
        # Alternating cheap/absorbing stages (VT_ALT16=1; the no-final-metric kernel of the cheap
        # form): body stages C A C A C A instead of N C A N C A -- every even stage is a cheap
        # stage (one VIADDMNMX per state, metrics leave it offset by -S(p0)), every odd stage
        # absorbs the offsets through combos.  The renormalisation moves into the absorbing
        # stages 3 and 5 (a cheap stage cannot fold it), by the minimum over a state set T taken
        # two stages earlier (after stages 1 and 3, clean values): metrics then stay in
        # [Sb', Sb' + Delta + 2560 + ...] with Sb' = 256 W_T + 2*dmax (renorm_set with W_T <= 8).
        self.alt = os.environ.get("VT_ALT16", "0") == "1" and self.cheap and self.B == 2 and not tc and not mma
        self.alt_now = False
        if self.alt:
            r = renorm_set(K, gens, 8)
            assert r is not None, "alternating form: no renormalisation set"
            self.alt_T, w_t = r
            self.Sb_alt = 256 * w_t + 2 * self.dmax
            assert self.Sb_alt + delta + 2560 + 512 < (1 << (16 - self.L)), "alternating form: metric range"

        self.polfrac = os.environ.get("VT_POLFRAC16", "")  # e.g. "0.75": fractional evict_last/evict_first
        if self.polfrac:
            self.EF = 0
        # Traceback ring depth (groups prefetched ahead): 4.  8 (fits two CTAs per SM for K=7
        # r1/2) measured 165.2 vs 167.4 Gbps at 2^20 windows, 123.5 vs 120.0 at 2^16 (the
        # CTA's last-tile traceback is latency-bound) -- VT_TBD16 overrides.
        if not tc and "VT_TBD16" in os.environ:
            self.TBD = int(os.environ["VT_TBD16"])
            assert self.TBD in (2, 4, 8, 16)
        ring = self.TBD * (self.S // 16)
        # row stride (uint4) of the per-thread LLR rows: odd, so the realignment's 4-byte loads
        # (the same byte offset in every thread's row) spread over 8 bank groups (4-way) instead
        # of 4 (NL = 6: 8-way) or 1 (NL = 8: 32-way)
        self.RS = self.NL | 1 if self.pbr else self.NL
        self.SMEM = (4 * self.RS + ring) * NT * 16  # dynamic shared memory bytes
        if self.tma:  # the TMA barriers after the rows (keeps the rows' alignment)
            self.SMEM_TMA_OFF = self.SMEM
            self.SMEM += 16 * (NT // 32)
        if self.tmh:
            self.SMEM_TM_OFF = self.SMEM  # TMEM allocation result
            self.SMEM += 16

        # tensor-core branch metrics (paper formulation): int8 LLR tile x +-8 codeword matrix
        self.tc = tc
        # mma.sync register-fragment branch metrics (the 16x2mma form, see mma_block): per body and
        # warp, 12 mma.sync.m16n8k16 s8 of the realigned LLR words against the +-8 codeword matrix;
        # A fragments through a transposed shared-memory tile, D fragments back to the owning
        # threads with stmatrix; per warp 8 x 33 + 32 x 32 words of shared memory
        self.mma = mma
        if mma:
            assert self.cheap and self.B == 2 and self.pbr and NT == 128 and self.P == 6
            self.MXOFF = self.SMEM
            self.MXW = (8 * 33 + 32 * 32) * 4
            self.SMEM += self.MXW * (NT // 32)
        # tc: rows-ready mbarrier instead of a CTA-wide __syncthreads before each MMA issue
        self.tc_mbar = tc and os.environ.get("VT_TC_SYNC", "mbar") == "mbar"
        if tc:
            assert self.cheap and self.B == 2 and self.CH * self.B <= 24 and NT == 128
            self.TCN = self.CH * 4           # MMA N: 4 pattern sums per stage of a chunk
            self.TCOFF = self.SMEM           # A tiles [buffer][window set] 4 KB each, B 2 KB, barriers
            self.SMEM += 4 * 4096 + 2048 + 64

    def cheap_candidate(self) -> bool:
        """K=7 rate 1/2 (the cheap-middle-stage form): the evict-first history split helps it
        (+0.9%) and costs K=7 r1/3 0.7%."""
        return self.B == 2 and self.K == 7

    def pattern(self, i: int, u: int) -> int:
        reg = (u << self.k) | i
        return sum(parity(g & reg) << b for b, g in enumerate(self.gens))

    def emit(self, s: str = "") -> None:
        self.lines.append(s)

    def emit_S(self, ind: str, q: int, pats) -> None:
        """Pattern sums S_p = sum_b (U or N)_b of body stage q for the patterns `pats`:
        from the U/N terms, or (tc variant) from the chunk's tensor-core contraction
        in TMEM (one 32x32b.x4 load per window set: the 4 pattern columns of the stage)."""
        e = self.emit
        pats = sorted(set(pats))
        if self.mma:
            if q % 2 == 0:
                self.mma_block(ind, q // 2)
            return
        if not self.tc:
            for p in pats:
                expr = " + ".join(f"{'N' if (p >> b) & 1 else 'U'}{q}_{b}" for b in range(self.B))
                e(f"{ind}const uint32_t S{q}_{p} = {expr};")
            return
        # the loads of body stage q are issued during stage q-1 (stage 0 loads for itself),
        # so tcgen05.wait::ld rarely waits
        if q == 0:
            self.tc_load(ind, 0)
        e(f"{ind}vt::tc::wait_ld();")
        for p in pats:  # window A in the low half, window B in the high half
            e(f"{ind}const uint32_t S{q}_{p} = vt::prmt(ta{q}_{p}, tb{q}_{p}, 0x5410u);")
        if q + 1 < self.P:
            self.tc_load(ind, q + 1)

    def mma_block(self, ind: str, sp: int) -> None:
        """Pattern sums of body stages 2sp, 2sp+1 on the tensor cores (mma.sync, SURVEY.md:270-273).
        Tile m (m = 0..3) of the warp's 64 windows: row g = window A and row g+8 = window B of
        lane 4g+m; D[row][n] = 2048 + sum_k llr[row][k] * W[k][n] = S_p of stage 2sp + n/4,
        p = n%4 (W = +-8 codeword entries: the kernel's U/N scaling, module docstring).  Lane
        (g,q) gets columns 2q, 2q+1 of its quad's rows; PRMT packs windows A/B into 16x2 words
        (X: even columns, Y: odd) and stmatrix writes them as rows of the owning lanes' tiles, so
        after a __syncwarp each lane reads its 8 words with two 16-byte loads."""
        e = self.emit
        e(f"{ind}uint32_t mX{sp}[4], mY{sp}[4];")
        e(f"{ind}#pragma unroll")
        e(f"{ind}for (int m = 0; m < 4; ++m) {{")
        e(f"{ind}  uint32_t d0, d1, d2, d3;")
        e(f"{ind}  vt::mx::mma_s8_16816(d0, d1, d2, d3, ma0[m], ma1[m], mb{sp}, 2048u);")
        e(f"{ind}  mX{sp}[m] = vt::prmt(d0, d2, 0x5410u);")
        e(f"{ind}  mY{sp}[m] = vt::prmt(d1, d3, 0x5410u);")
        e(f"{ind}}}")
        e(f"{ind}vt::mx::stmatrix_x4(mst0 + mstc({sp}, 0), mX{sp}[0], mY{sp}[0], mX{sp}[1], mY{sp}[1]);")
        e(f"{ind}vt::mx::stmatrix_x4(mst1 + mstc({sp}, 1), mX{sp}[2], mY{sp}[2], mX{sp}[3], mY{sp}[3]);")
        e(f"{ind}__syncwarp();")
        e(f"{ind}const uint4 mvx{sp} = *reinterpret_cast<const uint4*>(ys + mrd({2 * sp}));")
        e(f"{ind}const uint4 mvy{sp} = *reinterpret_cast<const uint4*>(ys + mrd({2 * sp + 1}));")
        q0, q1 = 2 * sp, 2 * sp + 1
        for nm, v in ((f"S{q0}_0", f"mvx{sp}.x"), (f"S{q0}_2", f"mvx{sp}.y"), (f"S{q1}_0", f"mvx{sp}.z"),
                      (f"S{q1}_2", f"mvx{sp}.w"), (f"S{q0}_1", f"mvy{sp}.x"), (f"S{q0}_3", f"mvy{sp}.y"),
                      (f"S{q1}_1", f"mvy{sp}.z"), (f"S{q1}_3", f"mvy{sp}.w")):
            e(f"{ind}const uint32_t {nm} = {v};")

    def mma_setup(self) -> None:
        """Per-lane constants of the 16x2mma form: B fragments (codeword matrix of each stage
        pair), stmatrix row addresses, the lane's own tile row; rows 3 and 7 of the transposed
        A tile are zero (bytes 12..15 of a body)."""
        e = self.emit
        e(f"  char* const s_mxw = reinterpret_cast<char*>(smem_dyn) + {self.MXOFF} + (tid >> 5) * {self.MXW};")
        e("  uint32_t* const xsT = reinterpret_cast<uint32_t*>(s_mxw);  // [8 words][33 lanes]: the body's LLR words")
        e("  char* const ys = s_mxw + 1056;  // [32 lanes][8 x 16 B]: the lanes' pattern sums")
        e("  const int mlane = tid & 31, mg = mlane >> 2, mq = mlane & 3;")
        e("  xsT[3 * 33 + mlane] = 0u;")
        e("  xsT[7 * 33 + mlane] = 0u;")
        e("  // B fragment of stage pair sp: rows k = 4q..4q+3 of column n = g (stage 2sp + n/4, pattern n%4):")
        e("  // +8 / -8 where byte k is LLR b of that stage and bit b of the pattern is 0 / 1")
        for sp in range(3):
            e(f"  uint32_t mb{sp} = 0u;")
            e("  #pragma unroll")
            e("  for (int i = 0; i < 4; ++i) {")
            e(f"    const int k = 4 * mq + i, st = {2 * sp} + (mg >> 2), p = mg & 3;")
            e("    const int v = ((k >> 1) == st) ? ((((p >> (k & 1)) & 1) != 0) ? -8 : 8) : 0;")
            e(f"    mb{sp} |= (uint32_t)(v & 0xFF) << (8 * i);")
            e("  }")
        e("  // tile rows: lane L's row at ys + 128 L, chunk c at ((c + f(L)) & 7) * 16 with")
        e("  // f(L) = 4 ((L >> 2) & 1) + (((L & 3) + (L >> 3)) & 3): conflict-free for the stmatrix")
        e("  // rows (lanes 4r + m) and for the owners' 16-byte loads (8 consecutive lanes)")
        e("  auto mf = [](int L) { return 4 * ((L >> 2) & 1) + (((L & 3) + (L >> 3)) & 3); };")
        e("  const int mfo = mf(mlane);")
        e("  auto mrd = [&](int c) { return mlane * 128 + (((c + mfo) & 7) << 4); };")
        e("  // stmatrix: lanes 8j + r address row r of matrix j = (X, Y) of tiles 2h + (j >> 1): owner 4r + 2h + (j >> 1)")
        e("  const int mL0 = 4 * (mlane & 7) + (mlane >> 4), mL1 = mL0 + 2;")
        e("  const uint32_t mst0 = vt::tc::smem_u32(ys) + mL0 * 128, mst1 = vt::tc::smem_u32(ys) + mL1 * 128;")
        e("  const int mf0 = mf(mL0) + ((mlane >> 3) & 1), mf1 = mf(mL1) + ((mlane >> 3) & 1);")
        e("  auto mstc = [&](int sp, int h) { return (uint32_t)((((2 * sp) + (h ? mf1 : mf0)) & 7) << 4); };")
        e("  uint32_t ma0[4], ma1[4];  // A fragments of the body (tiles m = 0..3)")

    def mma_body_a(self, ind: str) -> None:
        """A fragments of this body: every lane stores its realigned words into the transposed
        tile, then lane (g,q) loads word q of windows A/B of lanes 4g+m (m = 0..3)."""
        e = self.emit
        e(f"{ind}__syncwarp();  // the previous body's A-fragment loads are done")
        for k in range(3):
            e(f"{ind}xsT[{k} * 33 + mlane] = curA[{k}];")
            e(f"{ind}xsT[{4 + k} * 33 + mlane] = curB[{k}];")
        e(f"{ind}__syncwarp();")
        e(f"{ind}#pragma unroll")
        e(f"{ind}for (int m = 0; m < 4; ++m) {{")
        e(f"{ind}  ma0[m] = xsT[mq * 33 + 4 * mg + m];")
        e(f"{ind}  ma1[m] = xsT[(4 + mq) * 33 + 4 * mg + m];")
        e(f"{ind}}}")

    def tc_load(self, ind: str, q: int) -> None:
        e = self.emit
        e(f"{ind}uint32_t ta{q}_0, ta{q}_1, ta{q}_2, ta{q}_3, tb{q}_0, tb{q}_1, tb{q}_2, tb{q}_3;")
        e(f"{ind}vt::tc::ld4(tcA + {4 * q}u, ta{q}_0, ta{q}_1, ta{q}_2, ta{q}_3);")
        e(f"{ind}vt::tc::ld4(tcA + {4 * q + self.TCN}u, tb{q}_0, tb{q}_1, tb{q}_2, tb{q}_3);")

    def stage(self, ind: str, q: int, names: list[str], defer: list | None = None) -> list[str]:
        """One radix-2 stage (body position q) for both windows.

        Candidate i1 is formed with a plain 32-bit IMAD (FMA pipe): every per-half
        value stays inside [0, 2^16) (range argument in the module docstring), so a
        32-bit add of the integer-packed addend E32 = e_B * 2^16 + e_A is exact per
        half even when e_A < 0 (renormalisation stage).  Candidate i0 goes through
        the fused VIADDMNMX.U16x2 add, which wraps per half, so it takes the
        per-half (mod 2^16) form D16.  Off the renormalisation stage the two forms
        coincide (all halves >= 0)."""
        B, L, S = self.B, self.L, self.S
        gq = q % L
        flag = f"cflag{q - gq}"
        e = self.emit
        for b in range(B if not (self.tc or self.mma) else 0):
            byte = q * B + b
            w, k = byte >> 2, byte & 3
            sel = k | ((8 | k) << 4) | ((4 + k) << 8) | ((12 + k) << 12)
            # (l_A, l_B) as signed 16-bit halves -> U = (l + 128) << L, N = (128 - l) << L, both >= 0
            e(f"{ind}const uint32_t P{q}_{b} = vt::prmt(curA[{w}], curB[{w}], {sel:#x}u);")
            e(f"{ind}const uint32_t U{q}_{b} = vt::vadd2(P{q}_{b}, 0x00800080u) << {L};")
            e(f"{ind}const uint32_t N{q}_{b} = {(256 << L) * 0x10001:#x}u - U{q}_{b};")
        outs, body, need_d, need_e = [None] * S, [], set(), set()
        fw = 1 << gq  # tie-flag weight of this stage
        is_c = (q % 2 == 0) if self.alt_now else (self.cheap and gq == 1)
        is_a = (q % 2 == 1) if self.alt_now else (self.cheap and gq == 2)
        ks = list(range(S // 2))
        # (the interleaved cheap/absorbing pairs keep the natural butterfly order)
        interleaved = (q in (0, 1, 4, 5)) if self.alt_now else (self.cheap and gq in (1, 2))
        if self.seed and not interleaved:
            self.rng.shuffle(ks)
        order = [x for k in ks for x in (k, k + S // 2)]
        if is_c:
            # CHEAP stage: with the i0 branch metric as a per-state offset phi_j of the
            # stored metric (stored = true - S(p0(j))), the update needs no candidate add:
            #   stored_j = max(m_i1 + T_p0, m_i0),  T_p0 = S(~p0) - S(p0) + 2^1 * flag
            # (patterns of i0 and i1 are complementary).  One VIADDMNMX per state pair.
            allp = set()
            for j in order:
                u = j >> (self.k - 1)
                i0 = (j << 1) & (S - 1)
                p0 = self.pattern(i0, u)
                allp.add(p0)
                allp.add(p0 ^ ((1 << B) - 1))
                nm = f"x{q}_{j}"
                body.append(f"{ind}const uint32_t {nm} = vt::vaddmax2({names[i0 | 1]}, T{q}_{p0}, {names[i0]});")
                outs[j] = nm
            self.emit_S(ind, q, allp)
            full = (1 << B) - 1
            done = set()
            for p in sorted(allp):
                if p in done:
                    continue
                pc = p ^ full
                # per half mod 2^16: T_p = S_pc - S_p + 2f ; T_pc = -T_p + 4f
                e(f"{ind}const uint32_t T{q}_{p} = vt::vadd2(vt::vadd2(S{q}_{pc}, ~S{q}_{p}), (1u + {fw}u * {flag}) * 0x10001u);")
                e(f"{ind}const uint32_t T{q}_{pc} = vt::vadd2(~T{q}_{p}, (1u + {2 * fw}u * {flag}) * 0x10001u);")
                done |= {p, pc}
            if defer is not None:
                defer.extend(body)
            else:
                self.lines.extend(body)
            return outs
        if is_a:
            # offset stage after the cheap one: state i carries phi_i = S1(p0(i)), so the
            # addends are combos S1(class of the predecessor) + S2(branch pattern)
            q1 = q - 1
            combos_d, combos_e = set(), set()
            for j in order:
                u = j >> (self.k - 1)
                i0 = (j << 1) & (S - 1)
                i1 = i0 | 1
                c0 = (self.pattern((i0 << 1) & (S - 1), i0 >> (self.k - 1)), self.pattern(i0, u))
                c1 = (self.pattern((i1 << 1) & (S - 1), i1 >> (self.k - 1)), self.pattern(i1, u))
                combos_d.add(c0)
                combos_e.add(c1)
                nm = f"x{q}_{j}"
                body.append(f"{ind}const uint32_t {nm} = vt::vaddmax2({names[i0]}, D{q}_{c0[0]}_{c0[1]}, "
                            f"vt::mad_u32({names[i1]}, 1u, E{q}_{c1[0]}_{c1[1]}));")
                outs[j] = nm
            pb_all = sorted({c[1] for c in combos_d | combos_e})
            self.emit_S(ind, q, pb_all)
            for p in sorted({c[1] for c in combos_e}):
                e(f"{ind}const uint32_t Sf{q}_{p} = S{q}_{p} + {flag} * {(1 << gq) * 0x10001:#x}u;")
            if self.alt_now and q in (3, 5):
                # renormalisation folded into the combos: -R per half mod 2^16 for the fused
                # VIADDMNMX operand, as a packed integer for the IMAD operand (see stage())
                for p in sorted({c[1] for c in combos_d}):
                    e(f"{ind}const uint32_t SR{q}_{p} = vt::vadd2(S{q}_{p}, negRa{q});")
                for p in sorted({c[1] for c in combos_e}):
                    e(f"{ind}const uint32_t SfR{q}_{p} = Sf{q}_{p} + negEa{q};")
                for pa, pb in sorted(combos_d):
                    e(f"{ind}const uint32_t D{q}_{pa}_{pb} = vt::vadd2(S{q1}_{pa}, SR{q}_{pb});")
                for pa, pb in sorted(combos_e):
                    e(f"{ind}const uint32_t E{q}_{pa}_{pb} = S{q1}_{pa} + SfR{q}_{pb};")
            else:
                for pa, pb in sorted(combos_d):
                    e(f"{ind}const uint32_t D{q}_{pa}_{pb} = S{q1}_{pa} + S{q}_{pb};")
                for pa, pb in sorted(combos_e):
                    e(f"{ind}const uint32_t E{q}_{pa}_{pb} = S{q1}_{pa} + Sf{q}_{pb};")
            if defer is not None:
                # interleave with the deferred cheap stage (all-ALU) so both pipes stay fed:
                # offset-stage butterfly k and k+S/4 consume cheap butterflies 2k, 2k+1
                h = len(defer) // 2  # butterflies
                cheap_bf = [defer[2 * i: 2 * i + 2] for i in range(h)]
                off_bf = [body[2 * i: 2 * i + 2] for i in range(h)]
                for k in range(h // 2):
                    self.lines.extend(cheap_bf[2 * k] + cheap_bf[2 * k + 1])
                    self.lines.extend(off_bf[k] + off_bf[k + h // 2])
                defer.clear()
            else:
                self.lines.extend(body)
            return outs
        # butterfly order (j, j + S/2 share predecessors i0, i1): the old metrics die in pairs
        for j in order:
            u = j >> (self.k - 1)
            i0 = (j << 1) & (S - 1)
            i1 = i0 | 1
            p0, p1 = self.pattern(i0, u), self.pattern(i1, u)
            need_d.add(p0)
            need_e.add(p1)
            nm = f"x{q}_{j}"
            body.append(f"{ind}const uint32_t {nm} = vt::vaddmax2({names[i0]}, D{q}_{p0}, "
                        f"vt::mad_u32({names[i1]}, 1u, E{q}_{p1}));")
            outs[j] = nm
        if gq == 0:
            e(f"{ind}const uint32_t kE{q} = negE + {flag} * 0x10001u;")
        self.emit_S(ind, q, need_d | need_e)
        for p in sorted(need_d | need_e):
            if p in need_d:
                d = f"vt::vadd2(S{q}_{p}, negR)" if gq == 0 else f"S{q}_{p}"
                e(f"{ind}const uint32_t D{q}_{p} = {d};")
            if p in need_e:
                k = f"kE{q}" if gq == 0 else f"{flag} * {(1 << gq) * 0x10001:#x}u"
                e(f"{ind}const uint32_t E{q}_{p} = S{q}_{p} + {k};")
        self.lines.extend(body)
        return outs

    def alt_ref(self, ind: str, q: int, names: list[str]) -> None:
        """Alternating form: renormalisation reference from the clean outputs of absorbing
        stage q (the minimum over the state set alt_T), applied two stages later in the
        absorbing stage q + 2 (negRa / negEa: -R per half mod 2^16 and as a packed integer)."""
        L = self.L
        e = self.emit
        lm = (0xFFFF & ~((1 << L) - 1)) * 0x10001
        vals = [names[t] for t in self.alt_T]
        expr = vals[0]
        for v in vals[1:]:
            expr = f"vt::vmin2({expr}, {v})"
        e(f"{ind}const uint32_t ar{q} = ({expr}) & {lm:#x}u;")
        e(f"{ind}const uint32_t negRa{q + 2} = vt::vadd2(~vt::vadd2(ar{q}, {((-(self.Sb_alt << L)) & 0xFFFF) * 0x10001:#x}u), 0x00010001u);")
        e(f"{ind}const uint32_t negEa{q + 2} = {(self.Sb_alt << L) * 0x10001:#x}u - ar{q};")

    def tma_issue(self, ind: str, k: str) -> None:
        """Lane 0: TMA chunk `k` of the warp's A and B window sets into buffer (k & 1):
        box {16 B, RS lines, 32 rows} from the line of lane 0's window (rows = lanes,
        2*F*B bytes apart), completion on the warp's mbarrier of that buffer."""
        e = self.emit
        box = 16 * self.RS * 32
        e(f"{ind}{{")
        e(f"{ind}  const int kb = ({k}) & 1;")
        e(f"{ind}  vt::mbar_expect_tx(s_bar + 2 * warp + kb, {2 * box}u);")
        e(f"{ind}  vt::tma_load_rows(llrA(kb), &tmap, (int)((oA + (int64_t)CH * B * ({k})) >> 4), 0, s_bar + 2 * warp + kb);")
        e(f"{ind}  vt::tma_load_rows(llrB(kb), &tmap, (int)((oB + (int64_t)CH * B * ({k})) >> 4), 0, s_bar + 2 * warp + kb);")
        e(f"{ind}}}")

    TBD = 4  # traceback ring depth (groups prefetched ahead into shared memory)

    def tb_fetch(self, ind: str, grp: str, ring: str) -> None:
        """cp.async the whole history group `grp` (clamped to a stored group) of this
        thread's slot into ring entry `ring`, and commit (one commit per step)."""
        S, SQ = self.S, self.S // 16
        e = self.emit
        e(f"{ind}{{")
        self.fetch_group(ind + "  ", grp, f"s_tb + ({ring}) * {SQ * NT} + tid")
        e(f"{ind}  vt::cp_async_commit();")
        e(f"{ind}}}")

    def fetch_group(self, ind: str, grp: str, dst_expr: str) -> None:
        """Group `grp` (clamped to a stored group) of the traced tile into the per-thread ring
        entry at `dst`: cp.async from the HBM scratch slot, or (tmh) from the TMEM window --
        tcgen05.ld of the thread's 16 words + shared-memory stores (warp-uniform choice)."""
        SQ = self.S // 16
        e = self.emit
        dst = "dst"
        if self.tmh:
            e(f"{ind}uint4* const dst = {dst_expr};")
            e(f"{ind}const int tpos = txa + txs * max({grp}, a.b_lo);")
            e(f"{ind}if (tmw_tb && (unsigned)(tpos - tm_p0) < {self.TMW}u) {{")
            e(f"{ind}  uint32_t v[16];")
            e(f"{ind}  vt::tc::ld16(tm_lane + (uint32_t)(tpos - tm_p0) * 16u, v);")
            e(f"{ind}  vt::tc::wait_ld();")
            for q in range(SQ):
                e(f"{ind}  {dst}[{q * NT}] = make_uint4(v[{4 * q}], v[{4 * q + 1}], v[{4 * q + 2}], v[{4 * q + 3}]);")
            e(f"{ind}}} else {{")
            ii = ind + "  "
        else:
            ii = ind
        if self.tmh:
            e(f"{ii}const uint32_t xo = (uint32_t)tpos * {SQ * NT * 16}u;")
        else:
            e(f"{ii}const uint32_t xo = (uint32_t)(txa + txs * max({grp}, a.b_lo)) * {SQ * NT * 16}u;")
            e(f"{ii}uint4* const dst = {dst_expr};")
        for q in range(SQ):
            e(f"{ii}vt::cp_async16({dst} + {q * NT}, slotc + xo + {q * NT * 16}u, 16, 0);")
        if self.tmh:
            e(f"{ind}}}")

    def drain_entry(self, r: str) -> str:
        """Ring entry r (0..7) of the last-tile drain: 0-3 the traceback ring, 4-7 the LLR row
        buffers (free once the CTA's last forward pass is done)."""
        SQ = self.S // 16
        return f"(({r}) < 4 ? s_tb + ({r}) * {SQ * NT} : s_llr + (({r}) - 4) * {SQ * NT}) + tid"

    def drain_last_tile(self, ind: str) -> None:
        """Traceback of the CTA's last tile, alone after the forward passes: latency-bound on
        the history fetches, so it prefetches 8 groups deep (the 4-entry ring + 4 entries in
        the LLR row buffers) instead of 4.  The prefill left groups tbb..tbb-3 in entries 0-3."""
        S, SQ, L = self.S, self.S // 16, self.L
        fm = (1 << L) - 1
        e = self.emit
        e(f"{ind}__syncthreads();  // every warp is done with its LLR rows (entries 4-7 span all threads' rows)")
        e(f"{ind}for (int r = 4; r < 8; ++r) {{  // groups tbb-4 .. tbb-7 -> entries 4-7")
        self.fetch_group(ind + "  ", "tbb - r", self.drain_entry('r'))
        e(f"{ind}  vt::cp_async_commit();")
        e(f"{ind}}}")
        e(f"{ind}int dr = 0;  // drain ring entry of group tbb")
        e(f"{ind}while (tbb >= a.b_lo) {{")
        e(f"{ind}#pragma unroll")
        e(f"{ind}  for (int u = 0; u < 2; ++u) {{")
        e(f"{ind}    vt::cp_async_wait_group<7>();")
        e(f"{ind}    const char* const rs = reinterpret_cast<const char*>({self.drain_entry('dr')});")
        for w, side in (("A", 0), ("B", 16)):
            e(f"{ind}    {{")
            e(f"{ind}      const uint32_t j = tb{w}.j;")
            e(f"{ind}      const uint32_t wd = *reinterpret_cast<const uint32_t*>(rs + ((j & 48u) << {NTS}) + (j & 12u));")
            e(f"{ind}      const uint32_t h = (wd >> ((j & 3u) * {L}u + {side}u)) & {fm}u;")
            e(f"{ind}      tb{w}.acc = (tb{w}.acc << {L}) | (j >> {self.k - L});")
            e(f"{ind}      tb{w}.j = ((j << {L}) | h) & {S - 1}u;")
            e(f"{ind}      tb{w}.lo -= {L};")
            e(f"{ind}      --tb{w}.b;")
            e(f"{ind}    }}")
        e(f"{ind}    --tbb;")
        e(f"{ind}    {{")
        self.fetch_group(ind + "      ", "tbb - 7", self.drain_entry('dr'))
        e(f"{ind}      vt::cp_async_commit();")
        e(f"{ind}    }}")
        e(f"{ind}    dr = (dr + 1) & 7;")
        e(f"{ind}  }}")
        e(f"{ind}  tbA.settle(a);")
        e(f"{ind}  tbB.settle(a);")
        e(f"{ind}}}")

    def tb_step_both(self, ind: str, p: int = 0) -> None:
        """Traceback step of both windows of the previous tile (shared group counter
        tbb).  The whole history group is prefetched TBD steps ahead into a per-thread
        shared-memory ring (cp.async: no data dependency, so DRAM latency is covered
        by TBD group ends of ACS work); the dependent walk then only touches shared
        memory.  Branch-free."""
        L, S, SQ = self.L, self.S, self.S // 16
        e = self.emit
        fm = (1 << L) - 1
        e(f"{ind}{{  // traceback step (previous tile, both windows)")
        e(f"{ind}  vt::cp_async_wait_group<{self.TBD - 1}>();")
        e(f"{ind}  const char* const rs = reinterpret_cast<const char*>(s_tb + tbr * {SQ * NT} + tid);")
        # state j's 3-bit field: word j >> 2 of the group (uint4 j >> 4, word (j >> 2) & 3),
        # bit offset 3 * (j & 3) (+16 for window B)
        for w, side in (("A", 0), ("B", 16)):
            e(f"{ind}  {{")
            e(f"{ind}    const uint32_t j = tb{w}.j;")
            e(f"{ind}    const uint32_t wd = *reinterpret_cast<const uint32_t*>(rs + ((j & 48u) << {NTS}) + (j & 12u));")
            e(f"{ind}    const uint32_t h = (wd >> ((j & 3u) * {L}u + {side}u)) & {fm}u;")
            e(f"{ind}    tb{w}.acc = (tb{w}.acc << {L}) | (j >> {self.k - L});")
            e(f"{ind}    tb{w}.j = ((j << {L}) | h) & {S - 1}u;")
            e(f"{ind}    tb{w}.lo -= {L};")
            e(f"{ind}    --tb{w}.b;")
            e(f"{ind}  }}")
        e(f"{ind}  --tbb;")
        self.tb_fetch(ind + "  ", f"tbb - {self.TBD - 1}", "tbr")
        e(f"{ind}  tbr = (tbr + 1) & {self.TBD - 1};")
        e(f"{ind}}}")

    def group_end(self, ind: str, ge: int = 0) -> None:
        """Renormalisation, traceback steps, history fields -> scratch + clear.
        ge = index of this group end inside the loop body."""
        L, S = self.L, self.S
        e = self.emit
        hm = ((1 << L) - 1) * 0x10001
        lm = (0xFFFF & ~((1 << L) - 1)) * 0x10001
        e(f"{ind}// ---- group end")
        e(f"{ind}// renormalise the next group by Lambda_0 - S_b (per window half); from the fresh")
        e(f"{ind}// state-0 metric (history masked), so the chain overlaps the rest of the group end")
        if self.fm:
            e(f"{ind}offA += pendA;")
            e(f"{ind}offB += pendB;")
        if self.alt_now:
            e(f"{ind}{{  // (alternating form: renormalised inside the absorbing stages)")
        else:
            e(f"{ind}{{")
        if self.alt_now:
            pass
        elif self.xmin:  # per-half minimum over all states or over the set rset (history bits masked after)
            # ternary tree min(min(a, b), c): ptxas fuses each into one VIMNMX3.U16x2
            vals = [f"m{j}" for j in (self.rset if self.rset else range(S))]
            lvl = 0
            while len(vals) > 1:
                nxt = []
                i = 0
                while i < len(vals):
                    grp = vals[i:i + 3]
                    if len(grp) == 1:
                        nxt.append(grp[0])
                    else:
                        nm = f"mn{lvl}_{i // 3}"
                        expr = f"vt::vmin2({grp[0]}, {grp[1]})"
                        if len(grp) == 3:
                            expr = f"vt::vmin2({expr}, {grp[2]})"
                        e(f"{ind}  const uint32_t {nm} = {expr};")
                        nxt.append(nm)
                    i += 3
                vals, lvl = nxt, lvl + 1
            e(f"{ind}  const uint32_t r0 = {vals[0]} & {lm:#x}u;")
        else:
            e(f"{ind}  const uint32_t r0 = m0 & {lm:#x}u;")
        if not self.alt_now:
            e(f"{ind}  const uint32_t rr = vt::vadd2(r0, {((-(self.Sb << L)) & 0xFFFF) * 0x10001:#x}u);")
            e(f"{ind}  negR = vt::vadd2(~rr, 0x00010001u);  // -R per half, mod 2^16 (fused-add operand)")
            e(f"{ind}  negE = {(self.Sb << L) * 0x10001:#x}u - r0;  // -R as a packed integer (IMAD operand)")
        if self.fm:
            e(f"{ind}  pendA = (int64_t)((r0 & 0xFFFFu) >> {L}) - {self.Sb};")
            e(f"{ind}  pendB = (int64_t)(r0 >> {16 + L}) - {self.Sb};")
        e(f"{ind}}}")
        e(f"{ind}// one traceback step per window of the previous tile (fields prefetched two groups")
        e(f"{ind}// ahead: the 2^L candidate states of a group are consecutive)")
        tb_after = bool(self.seed) and self.rng.random() < 0.5
        if not tb_after:
            self.tb_step_both(ind, ge % 2)
        # xmin kernels (ALU-heavy: the clears are LOP3s): the fields of the first CLRI states
        # are taken before the store branch and those states are cleared with IMADs (FMA
        # pipe); GEBF: the whole group end (fields, packs, clears) unconditional, only the
        # stores under the branch.  Warm-up groups carry zero fields, so both are exact.
        pre = range(S) if (self.xmin and self.gebf) else range(self.clri if self.xmin else 0)
        e(f"{ind}{{  // group-end scope (fields h, packs hw)")
        for j in pre:
            e(f"{ind}const uint32_t h{j} = m{j} & {hm:#x}u;")
        words = []
        for w in range(S // 4):
            acc = f"h{4 * w}"
            for t in range(1, 4):
                acc = f"vt::mad_u32(h{4 * w + t}, {1 << (L * t)}u, {acc})"
            words.append(acc)
        if self.xmin and self.gebf:
            for w in range(S // 4):
                e(f"{ind}const uint32_t hw{w} = {words[w]};")
            words = [f"hw{w}" for w in range(S // 4)]
        e(f"{ind}if (gidx >= a.b_lo) {{")
        e(f"{ind}  const int gs = gidx - a.b_lo;")
        e(f"{ind}  uint4* const dst = slot + (size_t)(parity ? (a.nbs - 1 - gs) : gs) * {S // 16} * {NT};")
        if self.EF:
            if not self.efc:
                e(f"{ind}  const uint64_t pol_h = gs < ef_lim ? pol_first : pol_last;")
        if not (self.xmin and self.gebf):
            for j in range(S):
                if j not in pre:
                    e(f"{ind}  const uint32_t h{j} = m{j} & {hm:#x}u;")
        pol = ("pol_c" if self.efc else "pol_h") if self.EF else "pol_last"
        if self.tmh:
            e(f"{ind}  const uint32_t hwv[16] = {{{', '.join(words)}}};")
            e(f"{ind}  const int tpos = parity ? (a.nbs - 1 - gs) : gs;")
            e(f"{ind}  if (tmw && (unsigned)(tpos - tm_p0) < 16u) {{  // warp-uniform: the group goes to TMEM")
            e(f"{ind}    vt::tc::st16(tm_lane + (uint32_t)(tpos - tm_p0) * 16u, hwv);")
            e(f"{ind}  }} else {{")
            for g in range(S // 16):
                e(f"{ind}    vt::st_global_v4_hint(dst + {g * NT}, make_uint4(hwv[{4 * g}], hwv[{4 * g + 1}], hwv[{4 * g + 2}], hwv[{4 * g + 3}]), {pol});")
            e(f"{ind}  }}")
        else:
            for g in range(S // 16):
                ws = ", ".join(words[4 * g: 4 * g + 4])
                e(f"{ind}  vt::st_global_v4_hint(dst + {g * NT}, make_uint4({ws}), {pol});")
        if not self.xmin:  # IMAD clear (FMA pipe): the ALU pipe is the K=7 r1/2 bottleneck
            for j in range(S):
                e(f"{ind}  m{j} = vt::mad_u32(h{j}, 0xFFFFFFFFu, m{j});")
        e(f"{ind}}}")
        if self.xmin:  # r1/3: unconditional clears after the branch (LOP3; IMAD for the CLRI states)
            for j in range(S):
                if j < self.clri:
                    e(f"{ind}m{j} = vt::mad_u32(h{j}, 0xFFFFFFFFu, m{j});")
                else:
                    e(f"{ind}m{j} &= {lm:#x}u;")
        e(f"{ind}}}")
        if tb_after:
            self.tb_step_both(ind, ge % 2)
        e(f"{ind}++gidx;")

    def kernel(self) -> str:
        """Both variants: vtk16_<code> (tracks final metrics when a.final_metric is set)
        and vtk16nf_<code> (no final-metric bookkeeping: fewer live registers)."""
        self.lines = []
        e = self.emit
        e("// GENERATED by gen_kernels16.py -- do not edit.")
        e(f"// code {self.name}: K={self.K}, generators (octal) {', '.join(oct(g)[2:] for g in self.gens)}; "
          f"two windows per thread (16x2 halves), {self.L}-bit history groups, {self.P}-stage body, {self.CH}-stage chunks")
        e('#include "../vt_common.cuh"')
        e("")
        pre = "vtk16tc" if self.tc else ("vtk16mma" if self.mma else "vtk16")
        for fm in (True, False):
            self.fm = fm
            self.kernel_one(f"{pre}_{self.name}" if fm else f"{pre}nf_{self.name}")
        return "\n".join(self.lines)

    def kernel_one(self, name: str) -> None:
        K, B, S, L, P, CH, NL, NWC = self.K, self.B, self.S, self.L, self.P, self.CH, self.NL, self.NWC
        self.alt_now = self.alt and not self.fm  # (the final-metric kernel keeps N C A groups)
        SQ = S // 16  # uint4 of history words per group per thread
        e = self.emit
        targ = ", const __grid_constant__ CUtensorMap tmap" if self.tma else ""
        e(f'extern "C" __global__ void __launch_bounds__({NT}, {MINB16}) {name}(const vt::StreamArgs a{targ}) {{')
        nwc = "" if self.pbr else f", NWC = {NWC}"  # (NWC: chunk-wide realignment only)
        e(f"  constexpr int B = {B}, K = {K}, CH = {CH}, NL = {NL}{nwc};")
        e("  const int tid = threadIdx.x;")
        e(f"  // dynamic shared memory: LLR staging, 2 buffers (chunk parity) x 2 windows x NL uint4 per")
        e(f"  // thread (column layout), then the traceback ring: TBD x SQ uint4 per thread")
        e("  extern __shared__ __align__(16) uint4 smem_dyn[];")
        e("  uint4* const s_llr = smem_dyn;")
        e(f"  uint4* const s_tb = smem_dyn + {4 * self.RS * NT};  // (even GPB only)")
        e("  (void)s_tb;")
        if self.mma:
            self.mma_setup()
        if self.tmh:
            e("  // TMEM history window: positions [tm_p0, tm_p0 + 16) of the scratch slot (the middle:")
            e("  // every position holds an old group in one tile parity and a young one in the other)")
            e(f"  uint32_t* const tc_tm = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(smem_dyn) + {self.SMEM_TM_OFF});")
            e("  if (tid < 32) vt::tc::alloc<256>(tc_tm);")
            e("  vt::tc::fence_before();")
            e("  __syncthreads();")
            e("  vt::tc::fence_after();")
            e("  const uint32_t tm_lane = *tc_tm + ((uint32_t)(32 * (tid >> 5)) << 16);  // this warp's lane quarter")
            e("  const int tm_p0 = a.nbs >= 16 ? (a.nbs - 16) >> 1 : (1 << 30);")
            e("  bool tmw = false, tmw_tb = false;  // this warp's groups share one index (this tile / the traced one)")
        if self.polfrac:  # one fractional policy for every history store (no per-group select)
            e(f"  const uint64_t pol_last = VT_POLICY_LAST_FIRST({self.polfrac});")
        else:
            e("  const uint64_t pol_last = vt::policy_evict_last();")
        if self.EF:
            e("  const uint64_t pol_first = vt::policy_evict_first();")
        if self.EF:
            e(f"  const int ef_lim = (a.nbs * {self.EF}) >> 8;  // stored groups gs < ef_lim: evict-first")
        if self.tma:
            e(f"  uint64_t* const s_bar = reinterpret_cast<uint64_t*>(smem_dyn + {self.SMEM_TMA_OFF // 16});  // TMA chunk barriers [warp][buffer]")
            e("  const int warp = tid >> 5, lane = tid & 31;")
            e("  uint32_t tph = 0;  // phase parity of this warp's two barriers")
            e("  if (a.tma && lane == 0) {")
            e("    vt::mbar_init(s_bar + 2 * warp, 1);")
            e("    vt::mbar_init(s_bar + 2 * warp + 1, 1);")
            e("    vt::mbar_init_fence();")
            e("  }")
            e("  __syncwarp();")
        e("  const int64_t nwin = a.w1 - a.w0;")
        e("  const int64_t buf_bytes = (a.st1 - a.st0) * B;")
        e(f"  uint4* const slot = a.scratch + (size_t)blockIdx.x * a.nbs * {SQ} * {NT} + tid;")
        e("  // per-thread rows of NL*16 bytes: [buffer][window][thread]")
        e(f"  auto llrA = [&](int buf) {{ return reinterpret_cast<char*>(s_llr) + ((2 * buf) * {NT} + tid) * {16 * self.RS}; }};")
        e(f"  auto llrB = [&](int buf) {{ return reinterpret_cast<char*>(s_llr) + ((2 * buf + 1) * {NT} + tid) * {16 * self.RS}; }};")
        e(f"  vt::TracebackLite<K, {L}> tbA, tbB;")
        e("  tbA.running = tbB.running = false;")
        e("  tbA.j = tbB.j = 0u; tbA.acc = tbB.acc = 0ull; tbA.lo = tbB.lo = 0; tbA.b = tbB.b = -1;")
        e("  tbA.active = tbB.active = false;")
        e("  int parity = 0;")
        e("  int tbb = -1;  // next group of the previous tile to trace (both windows step in lockstep)")
        e("  int tbr = 0;   // traceback ring entry holding group tbb")
        e("  const char* const slotc = reinterpret_cast<const char*>(slot);")
        if self.tc:
            TCN = self.TCN
            e(f"  // ---- tensor-core branch metrics: per chunk, D[window][4*stage + pattern] = A . Bm with")
            e(f"  // A = the window's {2 * CH} int8 LLRs of the chunk (+ a bias byte), Bm = the +-8 codeword")
            e(f"  // matrix (+ bias row): S_p = 8 * sum_b (+-l_b) + 2048 = sum_b (U or N)_b  (tcgen05 kind::i8)")
            e(f"  char* const s_tc = reinterpret_cast<char*>(smem_dyn) + {self.TCOFF};")
            e("  uint64_t* const tc_bar = reinterpret_cast<uint64_t*>(s_tc + 4 * 4096 + 2048);")
            e("  uint32_t* const tc_tm = reinterpret_cast<uint32_t*>(s_tc + 4 * 4096 + 2048 + 16);")
            if self.tc_mbar:
                e("  uint64_t* const rows_bar = reinterpret_cast<uint64_t*>(s_tc + 4 * 4096 + 2048 + 32);  // rows ready")
            e(f"  for (int i = tid; i < {TCN} * 32; i += {NT}) {{")
            e("    const int n = i >> 5, k = i & 31, st = n >> 2, pp = n & 3;")
            e("    int v = 0;")
            e(f"    if (k < {2 * CH} && (k >> 1) == st) v = ((pp >> (k & 1)) & 1) ? -8 : 8;")
            e(f"    else if (k == {2 * CH}) v = 32;")
            e("    s_tc[4 * 4096 + vt::tc::kmaj(n, k)] = (char)v;")
            e("  }")
            e(f"  for (int i = tid; i < 4 * {NT}; i += {NT})  // A rows: bias byte 64 at k = {2 * CH}, zeros after")
            e(f"    *reinterpret_cast<uint2*>(s_tc + (i >> 7) * 4096 + vt::tc::kmaj(i & 127, {2 * CH})) = make_uint2(64u, 0u);")
            e("  if (tid < 32) vt::tc::alloc<256>(tc_tm);")
            e("  if (tid == 0) {")
            e("    vt::tc::mbar_init(tc_bar, 1);")
            e("    vt::tc::mbar_init(tc_bar + 1, 1);")
            if self.tc_mbar:
                e(f"    vt::tc::mbar_init(rows_bar, {NT});")
                e(f"    vt::tc::mbar_init(rows_bar + 1, {NT});")
            e('    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");')
            e("  }")
            e("  vt::tc::fence_proxy_async();")
            e("  vt::tc::fence_before();")
            e("  __syncthreads();")
            e("  vt::tc::fence_after();")
            e("  const uint32_t tmb = *tc_tm;")
            e("  const uint32_t tcrow = tmb + ((uint32_t)(32 * (tid >> 5)) << 16);  // this warp's TMEM lane quarter")
            e("  uint32_t tc_phase = 0;")
            e("  const uint64_t tc_db = vt::tc::desc_kmaj(vt::tc::smem_u32(s_tc + 4 * 4096));")
            e(f"  constexpr uint32_t TC_ID = vt::tc::idesc_i8({NT}, {TCN});")
            e("  // row tid of the chunk tiles (buffer buf): the realigned LLR words of windows A and B")
            e("  auto tc_write = [&](int buf, const uint32_t (&wa)[NWC], const uint32_t (&wb)[NWC]) {")
            e("    char* const ta = s_tc + (2 * buf) * 4096;")
            e("    char* const tb = ta + 4096;")
            e("    *reinterpret_cast<uint4*>(ta + vt::tc::kmaj(tid, 0)) = make_uint4(wa[0], wa[1], wa[2], wa[3]);")
            e("    *reinterpret_cast<uint2*>(ta + vt::tc::kmaj(tid, 16)) = make_uint2(wa[4], wa[5]);")
            e("    *reinterpret_cast<uint4*>(tb + vt::tc::kmaj(tid, 0)) = make_uint4(wb[0], wb[1], wb[2], wb[3]);")
            e("    *reinterpret_cast<uint2*>(tb + vt::tc::kmaj(tid, 16)) = make_uint2(wb[4], wb[5]);")
            e("  };")
            if self.tc_mbar:
                e("  // all rows written -> one thread issues the two MMAs of chunk buffer buf.  No CTA-wide")
                e("  // barrier: every thread arrives on the buffer's rows-ready mbarrier (count NT) and moves")
                e("  // on; only the issuing thread waits for the arrivals")
                e("  uint32_t rows_phase = 0;")
                e("  auto tc_issue = [&](int buf0, int nbuf) {")
                e("    vt::tc::fence_before();")
                e("    vt::tc::fence_proxy_async();")
                e("    for (int bb = buf0; bb < buf0 + nbuf; ++bb) vt::tc::mbar_arrive(rows_bar + bb);")
                e("    if (tid == 0) {")
                e("      for (int bb = buf0; bb < buf0 + nbuf; ++bb) {")
                e("        vt::tc::mbar_wait(rows_bar + bb, (rows_phase >> bb) & 1u);")
                e("        rows_phase ^= 1u << bb;")
                e("        vt::tc::fence_after();")
                e("        const uint32_t ab = vt::tc::smem_u32(s_tc + (2 * bb) * 4096);")
                e(f"        vt::tc::mma_i8(tmb + bb * 128, vt::tc::desc_kmaj(ab), tc_db, TC_ID);")
                e(f"        vt::tc::mma_i8(tmb + bb * 128 + {TCN}, vt::tc::desc_kmaj(ab + 4096), tc_db, TC_ID);")
                e("        vt::tc::commit(tc_bar + bb);")
                e("      }")
                e("    }")
                e("  };")
            else:
                e("  // all rows written -> one thread issues the two MMAs of chunk buffer buf")
                e("  auto tc_issue = [&](int buf0, int nbuf) {")
                e("    vt::tc::fence_before();")
                e("    vt::tc::fence_proxy_async();")
                e("    __syncthreads();")
                e("    if (tid == 0) {")
                e("      vt::tc::fence_after();")
                e("      for (int bb = buf0; bb < buf0 + nbuf; ++bb) {")
                e("        const uint32_t ab = vt::tc::smem_u32(s_tc + (2 * bb) * 4096);")
                e(f"        vt::tc::mma_i8(tmb + bb * 128, vt::tc::desc_kmaj(ab), tc_db, TC_ID);")
                e(f"        vt::tc::mma_i8(tmb + bb * 128 + {TCN}, vt::tc::desc_kmaj(ab + 4096), tc_db, TC_ID);")
                e("        vt::tc::commit(tc_bar + bb);")
                e("      }")
                e("    }")
                e("  };")
        e("  // history words of group grp: 4 states per 32-bit word (L bits each, +16 for window B);")
        e("  // traced tile: group grp sits at slot position x = txa + txs * grp (tiles alternate the order)")
        e("  int txa = -a.b_lo, txs = 1;  // (initial values keep the idle prefetches inside the slot)")
        e(f"  const int ng = a.nc * {CH // L};  // history groups per window")
        e(f"  for (int64_t tile = blockIdx.x; tile * {2 * NT} < nwin; tile += gridDim.x, parity ^= 1) {{")
        e(f"    const int64_t wa = tile * {2 * NT} + 2 * tid, wb = wa + 1;")
        e("    const bool actA = wa < nwin, actB = wb < nwin;")
        e(f"    const vt::Window gA = vt::window_geometry<{CH}>(a, a.w0 + (actA ? wa : nwin - 1));")
        e(f"    const vt::Window gB = vt::window_geometry<{CH}>(a, a.w0 + (actB ? wb : nwin - 1));")
        e("    const int64_t oA = (gA.g0 - a.st0) * B, oB = (gB.g0 - a.st0) * B;")
        e("    // the window's whole staged span (16-byte words) lies inside the buffer: unchecked copies")
        e(f"    const int64_t span = (int64_t)a.nc * CH * B + 16 * NL;")
        e("    const bool fastA = oA >= 0 && oA + span <= buf_bytes, fastB = oB >= 0 && oB + span <= buf_bytes;")
        if self.pbr:
            e("    // 32-bit per-chunk bookkeeping: misalignment base and front-padding stages of each window")
            e("    const int moA = (int)(oA & 15), moB = (int)(oB & 15);")
            e(f"    const int padA = (int)min(max(gA.s - gA.g0, (int64_t)0), (int64_t){1 << 20}), "
              f"padB = (int)min(max(gB.s - gB.g0, (int64_t)0), (int64_t){1 << 20});")
        m0 = (self.Sb << L) * 0x10001 if self.cheap else 0  # cheap stages need m_i1 + T >= 0 from the start
        if self.alt_now:
            m0 = (self.Sb_alt << L) * 0x10001
        e("    " + " ".join(f"uint32_t m{j} = {m0:#x}u;" for j in range(S)))
        e("    uint32_t negR = 0, negE = 0;")
        if self.fm:
            o0 = -self.Sb if self.cheap else 0
            e(f"    int64_t offA = {o0}, offB = {o0}, pendA = 0, pendB = 0;")
        if self.pbr:
            e(f"    uint32_t curA[{self.NWB}], curB[{self.NWB}];  // this body's LLR words (realigned per body)")
        elif not self.tc:
            e("    uint32_t curA[NWC], curB[NWC];")
        e("    // leading zero-LLR padding keeps all-zero metrics at zero: skip whole bodies of it")
        if self.tc or self.mma:  # warp-uniform: tcgen05.ld / mma.sync / stmatrix are .sync.aligned, so every lane must run the same bodies
            e(f"    const int it0 = (int)__reduce_min_sync(0xFFFFFFFFu, (unsigned)min(min(max(gA.s - gA.g0, (int64_t)0), "
              f"max(gB.s - gB.g0, (int64_t)0)) / {P}, (int64_t){self.CHB}));")
        else:
            e(f"    const int it0 = (int)min(min(max(gA.s - gA.g0, (int64_t)0), max(gB.s - gB.g0, (int64_t)0)) / {P}, "
              f"(int64_t){self.CHB});")
        e("    int it_start = it0;")
        if self.tmh:
            e("    tmw = __all_sync(0xFFFFFFFFu, it0 == __shfl_sync(0xFFFFFFFFu, it0, 0));")
        if self.tc:
            e(f"    const int64_t oA0 = oA + (int64_t)it0 * {P * B}, oB0 = oB + (int64_t)it0 * {P * B};")
        e("    // chunks are staged two ahead (cp.async groups): chunk k lives in buffer k & 1")
        if self.tma:
            e("    // TMA staging when every window of the warp is interior (uniform F*B stride) and")
            e("    // in the buffer: one box per window set and chunk, issued by lane 0")
            e("    const bool tmaw = a.tma && __all_sync(0xFFFFFFFFu, actA && actB && fastA && fastB);")
            e("    if (tmaw) {")
            e("      __syncwarp();  // every lane is done with the previous tile's rows")
            e("      if (lane == 0) {")
            e("        vt::fence_proxy_async_smem();")
            self.tma_issue("        ", "0")
            e("        if (a.nc > 1) {")
            self.tma_issue("          ", "1")
            e("        }")
            e("      }")
            e("      vt::mbar_wait_parity(s_bar + 2 * warp, tph & 1u);")
            e("      tph ^= 1u;")
            e("    } else {")
        ind = "      " if self.tma else "    "
        if self.pbr:
            e(f"{ind}vt::stage_row<NL>(llrA(0), a.llr, buf_bytes, oA, fastA);")
            e(f"{ind}vt::stage_row<NL>(llrB(0), a.llr, buf_bytes, oB, fastB);")
        else:
            e(f"{ind}vt::stage_row<NL>(llrA(0), a.llr, buf_bytes, oA0, fastA);")
            e(f"{ind}vt::stage_row<NL>(llrB(0), a.llr, buf_bytes, oB0, fastB);")
        e(f"{ind}if (a.nc > 1) {{")
        e(f"{ind}  vt::stage_row<NL>(llrA(1), a.llr, buf_bytes, oA + (int64_t)CH * B, fastA);")
        e(f"{ind}  vt::stage_row<NL>(llrB(1), a.llr, buf_bytes, oB + (int64_t)CH * B, fastB);")
        e(f"{ind}}}")
        e(f"{ind}vt::cp_async_commit();")
        e(f"{ind}vt::cp_async_wait_group<0>();")
        if self.tma:
            e("    }")
        zb0A = f"(int)min(max((gA.s - gA.g0 - (int64_t)it0 * {P}) * B, (int64_t)0), (int64_t)CH * B)"
        zb0B = f"(int)min(max((gB.s - gB.g0 - (int64_t)it0 * {P}) * B, (int64_t)0), (int64_t)CH * B)"
        if self.tc:
            e("    {  // chunks 0 and 1 -> tiles 0 and 1 -> MMAs into TMEM buffers 0 and 1")
            e("      uint32_t rA[NWC], rB[NWC];")
            e(f"      vt::realign_row<NWC>(rA, llrA(0), (int)(oA0 & 15), {zb0A});")
            e(f"      vt::realign_row<NWC>(rB, llrB(0), (int)(oB0 & 15), {zb0B});")
            e("      tc_write(0, rA, rB);")
            e("      if (a.nc > 1) {")
            e("        vt::realign_row<NWC>(rA, llrA(1), (int)((oA + (int64_t)CH * B) & 15), "
              "(int)min(max((gA.s - (gA.g0 + (int64_t)CH)) * B, (int64_t)0), (int64_t)CH * B));")
            e("        vt::realign_row<NWC>(rB, llrB(1), (int)((oB + (int64_t)CH * B) & 15), "
              "(int)min(max((gB.s - (gB.g0 + (int64_t)CH)) * B, (int64_t)0), (int64_t)CH * B));")
            e("        tc_write(1, rA, rB);")
            e("      }")
            e("      tc_issue(0, a.nc > 1 ? 2 : 1);")
            e("    }")
        e(f"    int gidx = it0 * {self.GPB};")
        e("    // traceback of the previous tile: one group step per forward group, loads one group ahead")
        e("    for (int c = 0; c < a.nc; ++c) {")
        if self.EF and self.efc:
            e(f"      // history L2 policy per chunk (CTA-uniform: no per-store uniform-register move)")
            e(f"      const uint64_t pol_c = (c * {self.CHB * self.GPB} - a.b_lo < ef_lim) ? pol_first : pol_last;")
        if self.tc:
            e("      const int64_t onA = oA + (int64_t)CH * B * (c + 1), onB = oB + (int64_t)CH * B * (c + 1);")
        if self.tc:
            e("      if (c + 2 < a.nc) {")
            e(f"        vt::stage_row_rel<NL>(llrA(c & 1), a.llr, buf_bytes, oA, CH * B * (c + 2), fastA);")
            e(f"        vt::stage_row_rel<NL>(llrB(c & 1), a.llr, buf_bytes, oB, CH * B * (c + 2), fastB);")
            e("      }")
        if self.tc:
            # (tc: chunk c+2 is realigned at the end of THIS chunk, which may run no traceback
            # step at all (leading-padding skip), so the staging needs its own commit group)
            e("      vt::cp_async_commit();")
        if self.tc:
            e("      vt::tc::mbar_wait(tc_bar + (c & 1), (tc_phase >> (c & 1)) & 1u);  // chunk c's branch metrics")
            e("      tc_phase ^= 1u << (c & 1);")
            e("      vt::tc::fence_after();")
            e("      uint32_t tcA = tcrow + (uint32_t)(c & 1) * 128u;  // TMEM column of the next body's stage 0")
        e("#pragma unroll 1")
        e(f"      for (int it = it_start; it < {self.CHB}; ++it) {{")
        if self.pbr:
            e("        // this body's LLR words straight from the staged row of chunk c")
            for w in ("A", "B"):
                e(f"        vt::realign_row_at<{self.NWB}>(cur{w}, llr{w}(c & 1), ((mo{w} + CH * B * c) & 15) + {P * B} * it, "
                  f"min(max((pad{w} - CH * c - {P} * it) * B, 0), {P * B}));")
            if self.mma:
                self.mma_body_a("        ")
        names = [f"m{j}" for j in range(S)]
        deferred: list = []
        for q in range(P):
            if q % L == 0:
                e("        // history codes only in groups whose decisions are stored (warm-up needs none)")
                e(f"        const uint32_t cflag{q} = (gidx >= a.b_lo) ? 1u : 0u;")
            # (alternating form: a cheap stage is deferred and interleaved with the absorbing stage
            # after it only inside a group -- stage 2 ends a group, stage 3 starts one)
            dq = (q in (0, 1, 4, 5)) if self.alt_now else (self.cheap and q % L in (1, 2))
            names = self.stage("        ", q, names, deferred if dq else None)
            if self.alt_now and q in (1, 3):
                self.alt_ref("        ", q, names)
            if q % L == L - 1:
                for j in range(S):
                    e(f"        m{j} = {names[j]};")
                names = [f"m{j}" for j in range(S)]
                self.group_end("        ", q // L)
        if self.tc:
            e(f"        tcA += {4 * P}u;")
        if self.CHB > 5:
            # the 64-bit traceback accumulator holds < 32 unwritten bits after a settle plus
            # 3 bits per step: settle at least every 5 bodies (10 steps), not only per chunk
            e(f"        if (it == {self.CHB // 2 - 1}) {{ tbA.settle(a); tbB.settle(a); }}")
        e("      }")
        e("      it_start = 0;")
        if LOCK == 1 and NT == 256 and not (self.tc or self.mma or self.tmh):
            e(f"      asm volatile(\"bar.sync %0, 64;\" :: \"r\"(1 + (warp & 3)) : \"memory\");  // VT_LOCK16: warp pair lockstep")
        elif LOCK == 2 and NT == 256 and not (self.tc or self.mma or self.tmh):
            e("      __syncthreads();  // VT_LOCK16=2: CTA lockstep")
        e("      tbA.settle(a);  // whole words of the previous tile's traceback")
        e("      tbB.settle(a);")
        if self.tc:
            e("      if (c + 2 < a.nc) {  // chunk c+2 -> tile (c & 1) -> MMA into TMEM buffer (c & 1)")
            e("        if (c == 0) vt::cp_async_wait_group<0>(); else vt::cp_async_wait_group<3>();")
            e("        uint32_t rA[NWC], rB[NWC];")
            e("        const int64_t o2A = onA + (int64_t)CH * B, o2B = onB + (int64_t)CH * B;")
            e("        vt::realign_row<NWC>(rA, llrA(c & 1), (int)(o2A & 15), "
              "(int)min(max((gA.s - (gA.g0 + (int64_t)CH * (c + 2))) * B, (int64_t)0), (int64_t)CH * B));")
            e("        vt::realign_row<NWC>(rB, llrB(c & 1), (int)(o2B & 15), "
              "(int)min(max((gB.s - (gB.g0 + (int64_t)CH * (c + 2))) * B, (int64_t)0), (int64_t)CH * B));")
            e("        tc_write(c & 1, rA, rB);")
            e("        tc_issue(c & 1, 1);")
            e("      }")
        else:
            if self.tma:
                e("      if (tmaw) {  // chunk c's rows are consumed: TMA chunk c+2 into its buffer")
                e("        if (c + 2 < a.nc) {")
                e("          __syncwarp();")
                e("          if (lane == 0) {")
                e("            vt::fence_proxy_async_smem();")
                self.tma_issue("            ", "c + 2")
                e("          }")
                e("        }")
                e("        if (c + 1 < a.nc) {  // chunk c+1 landed")
                e("          vt::mbar_wait_parity(s_bar + 2 * warp + ((c + 1) & 1), (tph >> ((c + 1) & 1)) & 1u);")
                e("          tph ^= 1u << ((c + 1) & 1);")
                e("        }")
                e("      } else {")
            ind = "        " if self.tma else "      "
            e(f"{ind}// chunk c's rows are consumed: stage chunk c+2 into its buffer (rides on the next")
            e(f"{ind}// traceback step's commit group, >= 4 steps before chunk c+2 starts)")
            e(f"{ind}if (c + 2 < a.nc) {{")
            e(f"{ind}  vt::stage_row_rel<NL>(llrA(c & 1), a.llr, buf_bytes, oA, CH * B * (c + 2), fastA);")
            e(f"{ind}  vt::stage_row_rel<NL>(llrB(c & 1), a.llr, buf_bytes, oB, CH * B * (c + 2), fastB);")
            e(f"{ind}}}")
            e(f"{ind}if (c + 1 < a.nc) vt::cp_async_wait_group<{self.TBD - 1}>();  // chunk c+1 landed")
            if self.tma:
                e("      }")
        e("    }")
        e("    // the previous tile's remaining traceback steps, then its unstored tail")
        e("    while (tbb >= a.b_lo) {")
        self.tb_step_both("      ", 0)
        self.tb_step_both("      ", 1)
        e("      tbA.settle(a);")
        e("      tbB.settle(a);")
        e("    }")
        e("    tbA.b = tbB.b = tbb;")
        e("    if (tbA.running) tbA.drain_unstored(a);")
        e("    if (tbB.running) tbB.drain_unstored(a);")
        e("    // final states: argmax per window, lowest index on ties (reference.py:138)")
        e("    uint32_t bestA = 0, bestB = 0;")
        for j in range(S):
            e(f"    bestA = max(bestA, ((m{j} & 0xFFFFu) << 8) | {S - 1 - j}u);")
            e(f"    bestB = max(bestB, ((m{j} >> 16) << 8) | {S - 1 - j}u);")
        e(f"    const uint32_t jA = {S - 1}u - (bestA & 0xFFu), jB = {S - 1}u - (bestB & 0xFFu);")
        if self.fm:
          e("    if (a.final_metric) {")
          e(f"      const int64_t bias = ((int64_t)a.nc * CH - (int64_t)it0 * {P}) * {self.dmax};")
          e(f"      if (actA) a.final_metric[wa] = (int64_t)(bestA >> {8 + L}) + offA - bias;")
          e(f"      if (actB) a.final_metric[wb] = (int64_t)(bestB >> {8 + L}) + offB - bias;")
          e("    }")
        e("    tbA.start(gA, jA, actA, ng, a.N);")
        e("    tbB.start(gB, jB, actB, ng, a.N);")
        e("    txa = parity ? a.nbs - 1 + a.b_lo : -a.b_lo;")
        e("    txs = parity ? -1 : 1;")
        e("    tbb = ng - 1;")
        e("    tbr = 0;")
        e("    // this tile's history stores (STG) must be visible before the ring prefill and the next")
        e("    // tile's traceback read them back with cp.async: without the fence a fetch issued right")
        e("    // after the last stores could return stale data (measured: nondeterministic words on")
        e("    // multi-tile launches)")
        e("    __threadfence();")
        if self.tmh:
            e("    vt::tc::wait_st();  // this tile's TMEM groups before they are read back")
            e("    tmw_tb = tmw;")
        for r in range(self.TBD):
            self.tb_fetch("    ", f"tbb - {r}", f"{r}")
        e("  }")
        e("  // traceback of the CTA's last tile")
        if self.DRAIN8:
            self.drain_last_tile("  ")
        else:
            e("  while (tbb >= a.b_lo) {")
            self.tb_step_both("    ", 0)
            self.tb_step_both("    ", 1)
            e("    tbA.settle(a);")
            e("    tbB.settle(a);")
            e("  }")
        e("  tbA.b = tbB.b = tbb;")
        e("  if (tbA.running) tbA.drain_unstored(a);")
        e("  if (tbB.running) tbB.drain_unstored(a);")
        if self.tc:
            e("  vt::tc::fence_before();")
            e("  __syncthreads();")
            e("  if (tid < 32) vt::tc::dealloc<256>(tmb);")
        if self.tmh:
            e("  vt::tc::fence_before();")
            e("  __syncthreads();")
            e("  if (tid < 32) vt::tc::dealloc<256>(*tc_tm);")
        e("}")
        e("")
