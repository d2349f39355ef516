#!/usr/bin/env python3
"""Generator for the multi-lane packed 16x2 ACS kernels (K=8, 9: 128 / 256 states).

The 16x2 form of gen_kernels16.py (state j of two windows per 32-bit register,
window A in the low half, B in the high half; VIADDMNMX.U16x2 + carry-free IMAD
per state pair; 3-bit survivor fields in the low bits of each half) with the
2^(K-1) states of a window pair spread over T = 2^tau lanes of a warp, 64 per
lane -- the register budget of the K=7 kernel.

* Lane partition (as the s32 kernels, gen_kernels.py): at a stage boundary with
  partition `lo`, lane t owns the states whose bits [lo, lo+tau) equal t; a
  radix-2 stage moves the partition down one bit, so P = K-1-tau stages (two
  3-bit history groups for K=9) run lane-locally before a shared-memory
  transpose returns it to the top bits.  The lane-dependent part of each branch
  pattern is a per-lane swap of the U/N terms (LOP3 select with a lane mask).
* Renormalisation by the per-half minimum over a small state set T living on
  one lane (gen_kernels16.renorm_set; one shuffle from that lane; round 1: the
  exact minimum, a per-lane VIMNMX3 tree + 2 shuffles): the metric spread of
  (753,561) is bounded by Delta = 256 x 13 and min_T is within 256 * W_T of the
  exact minimum, so Lambda in [0, Sb' + Delta + 3*512) fits 13 bits.
* Shared memory per CTA: LLR rows per window pair (each lane stages every T-th
  16-byte chunk; rows are read by all T lanes), the per-thread traceback ring
  (cp.async prefetch of whole history groups, 4 deep) and the transpose buffer.
* Traceback: lane 0 walks window A, lane 1 window B; state j of group g lives in
  lane (j >> lo_g) & (T-1), slot slot_of(j, lo_g), lo_g = the partition at that
  group's end, read from that lane's ring entry.
"""
from __future__ import annotations

import os

from gen_kernels import parity
from gen_kernels16 import MEASURED_SEEDS, Gen16, history_bits, renorm_set, spread_weight

NT = 128  # threads per CTA


class Gen16M(Gen16):
    TBD = 4

    def __init__(self, name: str, K: int, gens: tuple[int, ...], T: int):
        self.name = name
        self.K = K
        self.k = K - 1
        self.S = 1 << self.k
        self.gens = gens
        self.B = len(gens)
        self.T = T
        self.tau = T.bit_length() - 1
        assert 1 << self.tau == T and T > 1
        self.SL = self.S // T
        assert self.SL in (32, 64), "32 or 64 states per lane"
        self.SQ = self.SL // 16
        self.top = self.k - self.tau
        self.P = 3 * (self.top // 3)  # stages per body between transposes (whole 3-bit groups)
        self.L = 3
        assert self.P % self.L == 0, "body must hold whole 3-bit groups"
        self.GPB = self.P // self.L
        self.dmax = 128 * self.B
        delta = 256 * spread_weight(K, gens)
        self.xmin = True
        full = (1 << self.B) - 1
        comp = all(self.pattern(((j << 1) & (self.S - 1)) | 1, j >> (self.k - 1)) ==
                   self.pattern((j << 1) & (self.S - 1), j >> (self.k - 1)) ^ full
                   for j in range(self.S))
        self.cheap = (os.environ.get("VT_CHEAP16M", "0") == "1" and comp and self.B == 2)  # measured 31.1 vs 31.5 Gbps (K=9)
        self.Sb = 2 * self.dmax if self.cheap else 0
        # Subset minimum (round 2, gen_kernels16.renorm_set): at group end ge (partition
        # lo = top - L*(ge+1)) renormalise by the minimum over a state set T_ge that lives on
        # ONE lane (min over its slots there + one shuffle from that lane) instead of the
        # per-lane tree over all 64 slots + 2 xor shuffles.  K=9 (753,561): T = {0, 193} /
        # {0, 4}, W_T = 9 / 10, Sb' = 2560: 2560 + 3328 + 3*512 = 7424 < 8192.
        self.clri = int(os.environ.get("VT_CLRI16M", "32"))  # group end: IMAD clears (see group_end)
        self.EF = int(os.environ.get("VT_EF16M", "0"))  # evict-first split of the history stores (1/256)
        self.gebf = os.environ.get("VT_GEBF16M", "1") == "1"
        self.rsets = None
        self.GPB = self.P // self.L
        if os.environ.get("VT_RSET", "1") == "1":
            # (the cheap middle stage needs metrics >= 2*dmax at its input: Sb' = 256 W_T + 2*dmax)
            wmax = ((1 << (16 - self.L)) - 1 - delta - self.L * 2 * self.dmax - self.Sb) // 256
            found = []
            for ge in range(self.GPB):
                lo = self.top - self.L * (ge + 1)
                best = None
                for lane in range(T):
                    r = renorm_set(K, gens, wmax, allowed=[self.state_of(x, lane, lo) for x in range(self.SL)])
                    if r is not None and (best is None or (len(r[0]), r[1]) < (len(best[0]), best[1])):
                        best = (r[0], r[1], lane)
                found.append(best)
            if all(f is not None for f in found):
                self.rsets = found
                self.Sb += 256 * max(f[1] for f in found)
        # the 16-bit range must hold (with the exact minimum at worst); codes whose spread does
        # not fit (e.g. K=9 with three or four outputs) get the s32 kernels only (code_units)
        self.supported = self.Sb + delta + self.L * 2 * self.dmax < (1 << (16 - self.L))
        self.pbr = True
        self.tc = False
        self.mma = False
        self.CHB = int(os.environ.get("VT_CHB16M", "5"))  # 5-body chunks: one traceback settle per chunk (see Gen16)
        self.CH = self.P * self.CHB
        self.NWB = -(-self.P * self.B // 4)
        self.NL = -(-(15 + self.CH * self.B + 4) // 16)
        self.RS = self.NL | 1
        self.NPAIR = NT // T
        # transpose buffer (words) per window pair: lane group stride G, pair stride XS
        self.G = (1 << self.top) + 32 // T
        self.XS = T * self.G + 4
        self.SM_LLR = 4 * self.RS * self.NPAIR * 16
        self.SM_RING = self.TBD * self.SQ * NT * 16
        self.SM_X = self.NPAIR * self.XS * 4
        self.SMEM = self.SM_LLR + self.SM_RING + self.SM_X
        self.lines: list[str] = []
        # neutral emission choices (as Gen16's VT_SEED16): butterfly order of the full
        # stages, traceback step before/after the history store
        import random
        self.seed = int(os.environ.get("VT_SEED16M", str(MEASURED_SEEDS.get((K, tuple(gens)), 0))))
        self.rng = random.Random(self.seed)

    # state <-> (lane, slot) for a partition at bits [lo, lo+tau)
    def slot_of(self, s: int, lo: int) -> int:
        return ((s >> (lo + self.tau)) << lo) | (s & ((1 << lo) - 1))

    def state_of(self, r: int, t: int, lo: int) -> int:
        return ((r >> lo) << (lo + self.tau)) | (t << lo) | (r & ((1 << lo) - 1))

    def lane_mask(self, b: int, lo: int) -> str | None:
        """Mask register selecting the swapped U/N terms of output b for this lane at a
        stage whose input partition is `lo`: parity(g_b & (t << lo)) as -1/0."""
        g = self.gens[b]
        bits = [(g >> (lo + i)) & 1 for i in range(self.tau)]
        if not any(bits):
            return None
        return "lm" + "".join(str(x) for x in bits)

    def stage(self, ind: str, q: int, names: list[str], defer: list | None = None) -> list[str]:
        """Radix-2 stage q of the body on slot-indexed names (partition top - q in,
        top - q - 1 out); same instruction forms as Gen16.stage."""
        B, L, S, SL = self.B, self.L, self.S, self.SL
        gq = q % L
        lo_in = self.top - q
        lo_out = lo_in - 1
        flag = f"cflag{q - gq}"
        e = self.emit
        for b in range(B):
            byte = q * B + b
            w, kk = byte >> 2, byte & 3
            sel = kk | ((8 | kk) << 4) | ((4 + kk) << 8) | ((12 + kk) << 12)
            e(f"{ind}const uint32_t P{q}_{b} = vt::prmt(curA[{w}], curB[{w}], {sel:#x}u);")
            m = self.lane_mask(b, lo_in)
            if m is None:
                e(f"{ind}const uint32_t U{q}_{b} = vt::vadd2(P{q}_{b}, 0x00800080u) << {L};")
                e(f"{ind}const uint32_t N{q}_{b} = {(256 << L) * 0x10001:#x}u - U{q}_{b};")
            else:  # this lane's pattern bit b is flipped: swap U and N
                e(f"{ind}const uint32_t u{q}_{b} = vt::vadd2(P{q}_{b}, 0x00800080u) << {L};")
                e(f"{ind}const uint32_t n{q}_{b} = {(256 << L) * 0x10001:#x}u - u{q}_{b};")
                e(f"{ind}const uint32_t U{q}_{b} = (u{q}_{b} & ~{m}) | (n{q}_{b} & {m});")
                e(f"{ind}const uint32_t N{q}_{b} = (n{q}_{b} & ~{m}) | (u{q}_{b} & {m});")
        outs, body, need_d, need_e = [None] * SL, [], set(), set()
        ks = list(range(SL // 2))
        if self.seed and not (self.cheap and gq in (1, 2)):
            self.rng.shuffle(ks)
        order = [x for k in ks for x in (k, k + SL // 2)]
        full = (1 << B) - 1

        def preds(r):
            j = self.state_of(r, 0, lo_out)
            u = j >> (self.k - 1)
            i0 = (j << 1) & (S - 1)
            i1 = i0 | 1
            r0, r1 = self.slot_of(i0, lo_in), self.slot_of(i1, lo_in)
            assert self.state_of(r0, 0, lo_in) == i0 and self.state_of(r1, 0, lo_in) == i1
            return j, u, i0, i1, r0, r1

        if self.cheap and gq == 1:
            allp = set()
            for r in order:
                j, u, i0, i1, r0, r1 = preds(r)
                p0 = self.pattern(i0, u)
                allp |= {p0, p0 ^ full}
                nm = f"x{q}_{r}"
                body.append(f"{ind}const uint32_t {nm} = vt::vaddmax2({names[r1]}, T{q}_{p0}, {names[r0]});")
                outs[r] = nm
            self.emit_S(ind, q, allp)
            done = set()
            for p in sorted(allp):
                if p in done:
                    continue
                pc = p ^ full
                e(f"{ind}const uint32_t T{q}_{p} = vt::vadd2(vt::vadd2(S{q}_{pc}, ~S{q}_{p}), (1u + 2u * {flag}) * 0x10001u);")
                e(f"{ind}const uint32_t T{q}_{pc} = vt::vadd2(~T{q}_{p}, (1u + 4u * {flag}) * 0x10001u);")
                done |= {p, pc}
            if defer is not None:
                defer.extend(body)
            else:
                self.lines.extend(body)
            return outs
        if self.cheap and gq == 2:
            q1 = q - 1
            combos_d, combos_e = set(), set()
            for r in order:
                j, u, i0, i1, r0, r1 = preds(r)
                c0 = (self.pattern((i0 << 1) & (S - 1), i0 >> (self.k - 1)), self.pattern(i0, u))
                c1 = (self.pattern((i1 << 1) & (S - 1), i1 >> (self.k - 1)), self.pattern(i1, u))
                combos_d.add(c0)
                combos_e.add(c1)
                nm = f"x{q}_{r}"
                body.append(f"{ind}const uint32_t {nm} = vt::vaddmax2({names[r0]}, D{q}_{c0[0]}_{c0[1]}, "
                            f"vt::mad_u32({names[r1]}, 1u, E{q}_{c1[0]}_{c1[1]}));")
                outs[r] = nm
            self.emit_S(ind, q, sorted({c[1] for c in combos_d | combos_e}))
            for p in sorted({c[1] for c in combos_e}):
                e(f"{ind}const uint32_t Sf{q}_{p} = S{q}_{p} + {flag} * {(1 << gq) * 0x10001:#x}u;")
            for pa, pb in sorted(combos_d):
                e(f"{ind}const uint32_t D{q}_{pa}_{pb} = S{q1}_{pa} + S{q}_{pb};")
            for pa, pb in sorted(combos_e):
                e(f"{ind}const uint32_t E{q}_{pa}_{pb} = S{q1}_{pa} + Sf{q}_{pb};")
            if defer is not None:
                h = len(defer) // 2
                cheap_bf = [defer[2 * i: 2 * i + 2] for i in range(h)]
                off_bf = [body[2 * i: 2 * i + 2] for i in range(h)]
                for k in range(h // 2):
                    self.lines.extend(cheap_bf[2 * k] + cheap_bf[2 * k + 1])
                    self.lines.extend(off_bf[k] + off_bf[k + h // 2])
                defer.clear()
            else:
                self.lines.extend(body)
            return outs
        for r in order:
            j, u, i0, i1, r0, r1 = preds(r)
            p0, p1 = self.pattern(i0, u), self.pattern(i1, u)
            need_d.add(p0)
            need_e.add(p1)
            nm = f"x{q}_{r}"
            body.append(f"{ind}const uint32_t {nm} = vt::vaddmax2({names[r0]}, D{q}_{p0}, "
                        f"vt::mad_u32({names[r1]}, 1u, E{q}_{p1}));")
            outs[r] = nm
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

    def tb_fetch(self, ind: str, grp: str, ring: str) -> None:
        SQ = self.SQ
        e = self.emit
        e(f"{ind}{{")
        e(f"{ind}  const uint32_t xo = (uint32_t)(txa + txs * max({grp}, a.b_lo)) * {SQ * NT * 16}u;")
        e(f"{ind}  uint4* const dst = s_tb + ({ring}) * {SQ * NT} + tid;")
        for qq in range(SQ):
            e(f"{ind}  vt::cp_async16(dst + {qq * NT}, slotc + xo + {qq * NT * 16}u, 16, 0);")
        e(f"{ind}  vt::cp_async_commit();")
        e(f"{ind}}}")

    def tb_step(self, ind: str) -> None:
        """One traceback step of this lane's window (lane 0: A, lane 1: B; lanes >= 2
        walk a copy that writes nothing).  Group tbb's fields sit in the ring entry tbr
        of lane (j >> lo_g) & (T-1), lo_g = the partition at that group's end."""
        L, S, SQ, T, tau = self.L, self.S, self.SQ, self.T, self.tau
        e = self.emit
        assert self.GPB in (1, 2)
        lo_a = self.top - self.L  # partition at the end of a body's first group
        lo_b = self.top - 2 * self.L if self.GPB == 2 else lo_a  # ... and of its second
        e(f"{ind}{{  // traceback step (previous tile)")
        e(f"{ind}  vt::cp_async_wait_group<{self.TBD - 1}>();")
        e(f"{ind}  __syncwarp(pm);  // the pair's ring entries for group tbb have landed")
        e(f"{ind}  const uint32_t j = tb.j;")
        e(f"{ind}  const bool odd = {'tbb & 1' if self.GPB == 2 else 'false'};")
        e(f"{ind}  const uint32_t tl = odd ? ((j >> {lo_b}) & {T - 1}u) : ((j >> {lo_a}) & {T - 1}u);")
        e(f"{ind}  const uint32_t r = odd ? (((j >> {lo_b + tau}) << {lo_b}) | (j & {(1 << lo_b) - 1}u)) "
          f": (((j >> {lo_a + tau}) << {lo_a}) | (j & {(1 << lo_a) - 1}u));")
        e(f"{ind}  const uint32_t wd = *reinterpret_cast<const uint32_t*>(rsb + tbr * {SQ * NT * 16} + "
          f"(r >> 4) * {NT * 16} + tl * 16u + (r & 12u));")
        e(f"{ind}  tb.step((wd >> ((r & 3u) * {L}u + side)) & {(1 << L) - 1}u);")
        e(f"{ind}  __syncwarp(pm);  // read before any lane refills its entry")
        e(f"{ind}  --tbb;")
        self.tb_fetch(ind + "  ", f"tbb - {self.TBD - 1}", "tbr")
        e(f"{ind}  tbr = (tbr + 1) & {self.TBD - 1};")
        e(f"{ind}}}")

    def group_end(self, ind: str, ge: int = 0) -> None:
        L, SL, SQ = self.L, self.SL, self.SQ
        e = self.emit
        hm = ((1 << L) - 1) * 0x10001
        lm = (0xFFFF & ~((1 << L) - 1)) * 0x10001
        if self.rsets:
            e(f"{ind}// ---- group end: renormalise by the per-half minimum over the state set T (one lane)")
        else:
            e(f"{ind}// ---- group end: renormalise by the exact per-half minimum over all lanes")
        if self.fm:
            e(f"{ind}offA += pendA;")
            e(f"{ind}offB += pendB;")
        e(f"{ind}{{")
        if self.rsets:
            Tset, _, owner = self.rsets[ge]
            lo = self.top - L * (ge + 1)
            vals = [f"m{self.slot_of(x, lo)}" for x in Tset]
        else:
            vals = [f"m{r}" for r in range(SL)]
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
        e(f"{ind}  uint32_t mn = {vals[0]};")
        if self.rsets:  # T lives on lane `owner` of the pair at this partition
            e(f"{ind}  mn = __shfl_sync(pm, mn, {owner}, {self.T});  // T = {{{', '.join(map(str, Tset))}}}")
        else:
            for d in range(self.tau):
                e(f"{ind}  mn = vt::vmin2(mn, __shfl_xor_sync(pm, mn, {1 << d}));")
        e(f"{ind}  const uint32_t r0 = mn & {lm:#x}u;")
        e(f"{ind}  const uint32_t rr = vt::vadd2(r0, {((-(self.Sb << L)) & 0xFFFF) * 0x10001:#x}u);")
        e(f"{ind}  negR = vt::vadd2(~rr, 0x00010001u);")
        e(f"{ind}  negE = {(self.Sb << L) * 0x10001:#x}u - r0;")
        if self.fm:
            e(f"{ind}  pendA = (int64_t)((r0 & 0xFFFFu) >> {L}) - {self.Sb};")
            e(f"{ind}  pendB = (int64_t)(r0 >> {16 + L}) - {self.Sb};")
        e(f"{ind}}}")
        tb_after = bool(self.seed) and self.rng.random() < 0.5
        if not tb_after:
            self.tb_step(ind)
        # fields of the first CLRI slots before the store branch, those slots cleared with
        # IMADs (FMA pipe; the LOP3 clears load the ALU pipe); GEBF: fields and packs
        # unconditional, only the stores under the branch (warm-up fields are zero)
        pre = range(SL) if self.gebf else range(self.clri)
        e(f"{ind}{{  // group-end scope (fields h, packs hw)")
        for r in pre:
            e(f"{ind}const uint32_t h{r} = m{r} & {hm:#x}u;")
        words = []
        for w in range(SL // 4):
            acc = f"h{4 * w}"
            for t in range(1, 4):
                acc = f"vt::mad_u32(h{4 * w + t}, {1 << (L * t)}u, {acc})"
            words.append(acc)
        if self.gebf:
            for w in range(SL // 4):
                e(f"{ind}const uint32_t hw{w} = {words[w]};")
            words = [f"hw{w}" for w in range(SL // 4)]
        e(f"{ind}if (gidx >= a.b_lo) {{")
        e(f"{ind}  const int gs = gidx - a.b_lo;")
        if self.EF:
            e(f"{ind}  const uint64_t pol_h = gs < ef_lim ? pol_first : pol_last;")
        e(f"{ind}  uint4* const dst = slot + (size_t)(parity ? (a.nbs - 1 - gs) : gs) * {SQ} * {NT};")
        if not self.gebf:
            for r in range(SL):
                if r not in pre:
                    e(f"{ind}  const uint32_t h{r} = m{r} & {hm:#x}u;")
        for g in range(SQ):
            ws = ", ".join(words[4 * g: 4 * g + 4])
            e(f"{ind}  vt::st_global_v4_hint(dst + {g * NT}, make_uint4({ws}), {'pol_h' if self.EF else 'pol_last'});")
        e(f"{ind}}}")
        # clear unconditionally (warm-up groups carry no decision bits): no phi moves
        for r in range(SL):
            if r < self.clri:
                e(f"{ind}m{r} = vt::mad_u32(h{r}, 0xFFFFFFFFu, m{r});")
            else:
                e(f"{ind}m{r} &= {lm:#x}u;")
        e(f"{ind}}}")
        if tb_after:
            self.tb_step(ind)
        e(f"{ind}++gidx;")

    def exchange_write(self, ind: str, lo: int) -> None:
        """Transpose, write half: the pair's metrics in partition `lo` go to the transpose
        buffer at their top-partition positions (the s32 kernels' conflict-free layout,
        gen_kernels.Gen.exchange).  The next body starts with exchange_read, so no metric
        register is carried around the body loop (no register moves after LDS.128)."""
        top, G, SL = self.top, self.G, self.SL
        e = self.emit
        e(f"{ind}// transpose: partition [{lo},{lo + self.tau}) -> [{top},{top + self.tau})")
        e(f"{ind}__syncwarp(pm);")
        lowmask = (1 << top) - 1
        r = 0
        while r < SL:
            s0 = self.state_of(r, 0, lo)
            run = 1
            while r + run < SL and self.state_of(r + run, 0, lo) == s0 + run and run < 4:
                run += 1
            off = (s0 & lowmask) + G * (s0 >> top)
            if run == 4 and off % 4 == 0:
                e(f"{ind}*reinterpret_cast<uint4*>(xw + {off} + (t << {lo})) = "
                  f"make_uint4(m{r}, m{r + 1}, m{r + 2}, m{r + 3});")
                r += 4
            else:
                e(f"{ind}xw[{off} + (t << {lo})] = m{r};")
                r += 1

    def exchange_read(self, ind: str, decl: bool = True) -> None:
        """Transpose, read half: this lane's 64 top-partition slots (LDS.128)."""
        e = self.emit
        e(f"{ind}__syncwarp(pm);")
        for r in range(0, self.SL, 4):
            e(f"{ind}const uint4 v{r} = *reinterpret_cast<const uint4*>(xr + {r});")
        ty = "uint32_t " if decl else ""
        e(f"{ind}" + " ".join(f"{ty}m{r + i} = v{r}.{'xyzw'[i]};" for r in range(0, self.SL, 4) for i in range(4)))

    def kernel(self) -> str:
        self.lines = []
        e = self.emit
        e("// GENERATED by gen_kernels16m.py -- do not edit.")
        e(f"// code {self.name}: K={self.K}, generators (octal) {', '.join(oct(g)[2:] for g in self.gens)}; "
          f"two windows per lane group of {self.T} lanes (16x2 halves, {self.SL} states per lane), "
          f"3-bit history groups, {self.P}-stage body, {self.CH}-stage chunks")
        e('#include "../vt_common.cuh"')
        e("")
        for fm in (True, False):
            self.fm = fm
            self.kernel_one(f"vtk16m_{self.name}" if fm else f"vtk16mnf_{self.name}")
        return "\n".join(self.lines)

    def kernel_one(self, name: str) -> None:
        K, B, S, L, P, CH, NL, T, SL, SQ = (self.K, self.B, self.S, self.L, self.P, self.CH, self.NL, self.T,
                                            self.SL, self.SQ)
        NPAIR, RS = self.NPAIR, self.RS
        e = self.emit
        e(f'extern "C" __global__ void __launch_bounds__({NT}, 1) {name}(const vt::StreamArgs a) {{')
        e(f"  constexpr int B = {B}, K = {K}, CH = {CH}, NL = {NL};")
        e("  const int tid = threadIdx.x;")
        e(f"  const int t = tid & {T - 1}, pair = tid >> {self.tau};")
        e(f"  const unsigned pm = {(1 << T) - 1}u << (tid & {32 - T});  // this pair's lanes")
        e("  extern __shared__ __align__(16) uint4 smem_dyn[];")
        e("  // LLR rows per window pair [buffer][window][pair] (RS uint4 each), traceback ring")
        e("  // [entry][uint4][thread], transpose buffer [pair][XS words]")
        e("  char* const s_llr = reinterpret_cast<char*>(smem_dyn);")
        e(f"  uint4* const s_tb = reinterpret_cast<uint4*>(s_llr + {self.SM_LLR});")
        e(f"  uint32_t* const xw = reinterpret_cast<uint32_t*>(s_llr + {self.SM_LLR + self.SM_RING}) + pair * {self.XS};")
        e(f"  const uint32_t* const xr = xw + t * {self.G};")
        e(f"  const char* const rsb = reinterpret_cast<const char*>(s_tb + pair * {T});  // the pair's ring columns")
        e("  const uint64_t pol_last = vt::policy_evict_last();")
        if self.EF:  # the oldest EF/256 of the stored groups evict-first (as Gen16)
            e("  const uint64_t pol_first = vt::policy_evict_first();")
            e(f"  const int ef_lim = (a.nbs * {self.EF}) >> 8;")
        e("  const int64_t nwin = a.w1 - a.w0;")
        e("  const int64_t buf_bytes = (a.st1 - a.st0) * B;")
        e(f"  uint4* const slot = a.scratch + (size_t)blockIdx.x * a.nbs * {SQ} * {NT} + tid;")
        e(f"  auto llrA = [&](int buf) {{ return s_llr + ((2 * buf) * {NPAIR} + pair) * {16 * RS}; }};")
        e(f"  auto llrB = [&](int buf) {{ return s_llr + ((2 * buf + 1) * {NPAIR} + pair) * {16 * RS}; }};")
        # lane masks for the U/N swaps
        masks = set()
        for q in range(P):
            for b in range(B):
                m = self.lane_mask(b, self.top - q)
                if m:
                    masks.add(m)
        for m in sorted(masks):
            bits = m[2:]
            terms = [f"((t >> {i}) & 1)" for i, c in enumerate(bits) if c == "1"]
            e(f"  const uint32_t {m} = 0u - (uint32_t)({' ^ '.join(terms)});")
        e(f"  const uint32_t side = (t & 1) ? 16u : 0u;  // traced window: lane 0 A, lane 1 B")
        e(f"  vt::TracebackLite<K, {L}> tb;")
        e("  tb.running = false; tb.j = 0u; tb.acc = 0ull; tb.lo = 0; tb.b = -1; tb.active = false;")
        e("  int parity = 0;")
        e("  int tbb = -1, tbr = 0;")
        e("  const char* const slotc = reinterpret_cast<const char*>(slot);")
        e("  int txa = -a.b_lo, txs = 1;")
        e(f"  const int ng = a.nc * {CH // L};")
        e(f"  for (int64_t tile = blockIdx.x; tile * {2 * NPAIR} < nwin; tile += gridDim.x, parity ^= 1) {{")
        e(f"    const int64_t wa = tile * {2 * NPAIR} + 2 * pair, wb = wa + 1;")
        e("    const bool actA = wa < nwin, actB = wb < nwin;")
        e(f"    const vt::Window gA = vt::window_geometry<{CH}>(a, a.w0 + (actA ? wa : nwin - 1));")
        e(f"    const vt::Window gB = vt::window_geometry<{CH}>(a, a.w0 + (actB ? wb : nwin - 1));")
        e("    const int64_t oA = (gA.g0 - a.st0) * B, oB = (gB.g0 - a.st0) * B;")
        e(f"    const int64_t span = (int64_t)a.nc * CH * B + 16 * NL;")
        e("    const bool fastA = oA >= 0 && oA + span <= buf_bytes, fastB = oB >= 0 && oB + span <= buf_bytes;")
        e("    const int moA = (int)(oA & 15), moB = (int)(oB & 15);")
        e(f"    const int padA = (int)min(max(gA.s - gA.g0, (int64_t)0), (int64_t){1 << 20}), "
          f"padB = (int)min(max(gB.s - gB.g0, (int64_t)0), (int64_t){1 << 20});")
        m0 = (self.Sb << L) * 0x10001
        e("    __syncwarp(pm);  // the previous tile's final metrics are read")
        e(f"    for (int r = 0; r < {SL}; r += 4) *reinterpret_cast<uint4*>(xw + t * {self.G} + r) = make_uint4({m0:#x}u, {m0:#x}u, {m0:#x}u, {m0:#x}u);")
        e("    uint32_t negR = 0, negE = 0;")
        if self.fm:
            e(f"    int64_t offA = {-self.Sb}, offB = {-self.Sb}, pendA = 0, pendB = 0;")
        e(f"    uint32_t curA[{self.NWB}], curB[{self.NWB}];")
        e(f"    const int it0 = (int)min(min(max(gA.s - gA.g0, (int64_t)0), max(gB.s - gB.g0, (int64_t)0)) / {P}, "
          f"(int64_t){self.CHB});")
        e("    int it_start = it0;")
        e("    __syncwarp(pm);  // the previous tile's rows are consumed")
        e(f"    vt::stage_row_part<NL, {T}>(llrA(0), a.llr, buf_bytes, oA, fastA, t);")
        e(f"    vt::stage_row_part<NL, {T}>(llrB(0), a.llr, buf_bytes, oB, fastB, t);")
        e("    if (a.nc > 1) {")
        e(f"      vt::stage_row_part<NL, {T}>(llrA(1), a.llr, buf_bytes, oA + (int64_t)CH * B, fastA, t);")
        e(f"      vt::stage_row_part<NL, {T}>(llrB(1), a.llr, buf_bytes, oB + (int64_t)CH * B, fastB, t);")
        e("    }")
        e("    vt::cp_async_commit();")
        e("    vt::cp_async_wait_group<0>();")
        e("    __syncwarp(pm);")
        e(f"    int gidx = it0 * {self.GPB};")
        e("    for (int c = 0; c < a.nc; ++c) {")
        e("#pragma unroll 1")
        e(f"      for (int it = it_start; it < {self.CHB}; ++it) {{")
        for w in ("A", "B"):
            e(f"        vt::realign_row_at<{self.NWB}>(cur{w}, llr{w}(c & 1), ((mo{w} + CH * B * c) & 15) + {P * B} * it, "
              f"min(max((pad{w} - CH * c - {P} * it) * B, 0), {P * B}));")
        self.exchange_read("        ")
        names = [f"m{r}" for r in range(SL)]
        deferred: list = []
        for q in range(P):
            if q % L == 0:
                e(f"        const uint32_t cflag{q} = (gidx >= a.b_lo) ? 1u : 0u;")
            names = self.stage("        ", q, names, deferred if (self.cheap and q % L in (1, 2)) else None)
            if q % L == L - 1:
                for r in range(SL):
                    e(f"        m{r} = {names[r]};")
                names = [f"m{r}" for r in range(SL)]
                self.group_end("        ", q // L)
        self.exchange_write("        ", self.top - P)
        if self.CHB * self.GPB > 10:
            # the 64-bit traceback accumulator holds < 32 unwritten bits after a settle plus
            # 3 bits per step: settle at least every 10 steps, not only per chunk
            e(f"        if (it == {self.CHB // 2 - 1}) tb.settle(a);")
        e("      }")
        e("      it_start = 0;")
        e("      tb.settle(a);")
        e("      __syncwarp(pm);  // chunk c's rows are consumed by every lane of the pair")
        e("      if (c + 2 < a.nc) {")
        e(f"        vt::stage_row_part<NL, {T}>(llrA(c & 1), a.llr, buf_bytes, oA + (int64_t)CH * B * (c + 2), fastA, t);")
        e(f"        vt::stage_row_part<NL, {T}>(llrB(c & 1), a.llr, buf_bytes, oB + (int64_t)CH * B * (c + 2), fastB, t);")
        e("      }")
        e("      if (c + 1 < a.nc) {")
        e(f"        vt::cp_async_wait_group<{self.TBD - 1}>();  // chunk c+1 landed (this lane's part)")
        e("        __syncwarp(pm);")
        e("      }")
        e("    }")
        e("    // the previous tile's remaining traceback steps, then its unstored tail")
        e("    while (tbb >= a.b_lo) {")
        self.tb_step("      ")
        self.tb_step("      ")
        e("      tb.settle(a);")
        e("    }")
        e("    tb.b = tbb;")
        e("    if (tb.running) tb.drain_unstored(a);")
        e("    // final states: argmax per window over all lanes, lowest index on ties (reference.py:138)")
        self.exchange_read("    ")
        e("    uint32_t bestA = 0, bestB = 0;")
        for r in range(SL):
            st = self.state_of(r, 0, self.top)
            e(f"    bestA = max(bestA, ((m{r} & 0xFFFFu) << 8) | ({S - 1 - st}u - ((uint32_t)t << {self.top})));")
            e(f"    bestB = max(bestB, ((m{r} >> 16) << 8) | ({S - 1 - st}u - ((uint32_t)t << {self.top})));")
        for d in range(self.tau):
            e(f"    bestA = max(bestA, __shfl_xor_sync(pm, bestA, {1 << d}));")
            e(f"    bestB = max(bestB, __shfl_xor_sync(pm, bestB, {1 << d}));")
        e(f"    const uint32_t jA = {S - 1}u - (bestA & 0xFFu), jB = {S - 1}u - (bestB & 0xFFu);")
        if self.fm:
            e("    if (a.final_metric && t == 0) {")
            e(f"      const int64_t bias = ((int64_t)a.nc * CH - (int64_t)it0 * {P}) * {self.dmax};")
            e(f"      if (actA) a.final_metric[wa] = (int64_t)(bestA >> {8 + L}) + offA - bias;")
            e(f"      if (actB) a.final_metric[wb] = (int64_t)(bestB >> {8 + L}) + offB - bias;")
            e("    }")
        e("    if (t & 1) tb.start(gB, jB, actB && t < 2, ng, a.N);")
        e("    else tb.start(gA, jA, actA && t < 2, ng, a.N);")
        e("    txa = parity ? a.nbs - 1 + a.b_lo : -a.b_lo;")
        e("    txs = parity ? -1 : 1;")
        e("    tbb = ng - 1;")
        e("    tbr = 0;")
        e("    // this tile's history stores (STG) must be visible before the ring prefill and the next")
        e("    // tile's traceback read them back with cp.async -- same thread and, for the traceback")
        e("    // lanes, other lanes of the pair: without the fence a fetch issued right after the last")
        e("    // stores could return stale data (measured: nondeterministic words on multi-tile launches)")
        e("    __threadfence();")
        e("    __syncwarp(pm);")
        for r in range(self.TBD):
            self.tb_fetch("    ", f"tbb - {r}", f"{r}")
        e("  }")
        e("  // traceback of the CTA's last tile")
        e("  while (tbb >= a.b_lo) {")
        self.tb_step("    ")
        self.tb_step("    ")
        e("    tb.settle(a);")
        e("  }")
        e("  tb.b = tbb;")
        e("  if (tb.running) tb.drain_unstored(a);")
        e("}")
        e("")
