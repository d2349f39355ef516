#!/usr/bin/env python3
"""Generate straight-line sm_100a ACS kernels, one per convolutional code.

Why a generator: the add-compare-select recursion for 2^(K-1) states is ~130
independent integer ops per thread per stage.  Written as C++ loops over
register arrays, NVVM needs minutes per kernel and ~2x the registers; emitted
as straight-line SSA code it compiles in about a second and ptxas sees exactly
the intended dataflow: IMAD.IADD on the FMA pipe feeding one DPX VIADDMNMX on
the ALU pipe per state-stage.

Reference semantics implemented (pkg/src/vitertile):
  * reference.py:60-83  predecessors i0 = 2*(j mod 2^(K-2)), i1 = i0+1, input u = j >> (K-2)
  * codes.py:183-193    branch output bit b = parity(g_b & ((u << (K-1)) | i))
  * reference.py:86-92,119-120  branch metric = sum_b (1 - 2*bit_b) * llr_b (maximised)
  * reference.py:121    tie -> second predecessor: the i1 candidate carries +2^p in the
                        low history bits, so signed max picks it on equal metrics
  * reference.py:124-125 renormalisation (exact): -lambda_0 folded into the branch metrics
  * reference.py:138    final state = lowest-index argmax
  * framing.py:68-141   windows / emit ranges (vt_common.cuh)

Loop structure.  The inner body is P = K-1 stages: after K-1 radix-2 stages
the state->register naming returns to the identity, so the loop back-edge
needs no register moves, and the body (~6 stages of code for K=7) stays small
enough for the instruction cache.  A history block is NIT = floor(16/P)
bodies (BL = P*NIT <= 16 stages, 12 for K=7): each state's low 16 bits record
the survivor-path decisions of the block and are streamed out at block end.

Threads per window T: K <= 7 keeps all 2^(K-1) metrics in one thread (T=1).
K = 8, 9 spread them over T = 2, 4 lanes.  Lanes are partitioned by tau =
log2(T) state bits starting at the top; a radix-2 stage maps a partition at
bits [lo, lo+tau) onto [lo-1, lo-1+tau) with no exchange, so P = K-1-tau
stages run exchange-free and one shared-memory transpose restores the top-bit
partition at the end of each body.  The lane-dependent part of the branch
parity is a per-lane LLR sign flip, so all lanes execute identical code.
"""
from __future__ import annotations

import argparse
import os

STANDARD_CODES = {
    # name: (K, generators as octal strings) -- BASELINE.json configs + tests/conftest.py:7-15
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

NT = 128  # threads per CTA


def parity(x: int) -> int:
    return bin(x).count("1") & 1


def threads_per_window(K: int) -> int:
    return {8: 2, 9: 4}.get(K, 1)


class Gen:
    def __init__(self, name: str, K: int, gens: tuple[int, ...], T: int):
        self.name = name
        self.K = K
        self.k = K - 1
        self.S = 1 << self.k
        self.gens = gens
        self.B = len(gens)
        self.T = T
        self.tau = T.bit_length() - 1
        assert 1 << self.tau == T
        self.SL = self.S // T
        self.SQ = max(self.SL // 8, 1)  # uint4 groups of histories per lane per block
        self.P = self.k - self.tau  # stages per loop body (register naming / lane partition period)
        self.NIT = 16 // self.P  # loop bodies per 16-stage history block
        self.R = 16 - self.P * self.NIT  # tail stages after the loop (their naming permutation is
        self.BL = 16  # absorbed by the block-end clears)
        self.top = self.k - self.tau if self.tau else 0
        self.G = (1 << self.top) + 32 // T if T > 1 else 0  # exchange buffer: lane-group stride (words)
        self.XS = T * self.G + 4 if T > 1 else 0  # exchange buffer: window stride (words)
        self.NL = self.B + 1  # staged 16-byte LLR words per block
        self.NWC = -(-self.BL * self.B // 4)  # realigned LLR words per block
        assert self.NWC + 4 <= 4 * self.NL
        # shared memory: LLR staging, traceback fields, lane exchange; above the 48 KB of
        # static shared memory a kernel may declare, the same layout goes dynamic
        smem = self.NL * NT * 16 + NT * 4 + ((NT // T) * self.XS * 4 if T > 1 else 0)
        self.dyn_smem = smem > 48 * 1024
        self.SMEM_DYN = smem if self.dyn_smem else 0
        self.lines: list[str] = []

    # -- state <-> (lane, slot) maps for a partition at bits [lo, lo+tau) --------
    def slot_of(self, s: int, lo: int) -> int:
        if self.tau == 0:
            return s
        return ((s >> (lo + self.tau)) << lo) | (s & ((1 << lo) - 1))

    def state_of(self, r: int, t: int, lo: int) -> int:
        if self.tau == 0:
            return r
        return ((r >> lo) << (lo + self.tau)) | (t << lo) | (r & ((1 << lo) - 1))

    def pattern(self, i: int, u: int) -> int:
        reg = (u << self.k) | i
        return sum(parity(g & reg) << b for b, g in enumerate(self.gens))

    def emit(self, s: str = ""):
        self.lines.append(s)

    # -- one body of `n` stages ------------------------------------------------
    def body(self, ind: str, n: int, names: list[str], lo: int, pfx: str, code_expr) -> tuple[list[str], int]:
        """Emit n stages reading metrics `names` in partition `lo`.  code_expr(q)
        returns the C expression of the history code added to the i1 candidate
        at body stage q.  Returns (output names, output partition)."""
        B = self.B
        cur = list(names)
        for q in range(n):
            lo_out = lo - 1 if self.tau else lo
            for b in range(B):
                byte = q * B + b
                expr = f"vt::llr_hi16(cur[{byte >> 2}], {byte & 3}u)"
                if self.T > 1:
                    expr = f"{expr} * f{self.top - lo}_{b}"
                self.emit(f"{ind}const int32_t {pfx}L{q}_{b} = {expr};")
            body, need_d, need_e = [], set(), set()
            outs = []
            for r in range(self.SL):
                j = self.state_of(r, 0, lo_out)
                u = j >> (self.k - 1)
                i0 = (j << 1) & (self.S - 1)
                i1 = i0 | 1
                r0, r1 = self.slot_of(i0, lo), self.slot_of(i1, lo)
                if self.tau:
                    assert self.state_of(r0, 0, lo) == i0 and self.state_of(r1, 0, lo) == i1
                p0, p1 = self.pattern(i0, u), self.pattern(i1, u)
                need_d.add(p0)
                need_e.add(p1)
                nm = f"{pfx}x{q}_{r}"
                body.append(f"{ind}const int32_t {nm} = vt::addmax({cur[r0]}, {pfx}D{q}_{p0}, "
                            f"vt::add_fma({cur[r1]}, {pfx}E{q}_{p1}));")
                outs.append(nm)
            for p in sorted(need_d | need_e):
                terms = [f"{'-' if (p >> b) & 1 else '+'} {pfx}L{q}_{b}" for b in range(B)]
                expr = " ".join(terms).lstrip("+ ")
                if q == 0:
                    expr = f"{expr} - rfold"
                self.emit(f"{ind}const int32_t {pfx}D{q}_{p} = {expr};")
                if p in need_e:
                    self.emit(f"{ind}const int32_t {pfx}E{q}_{p} = {code_expr(q, f'{pfx}D{q}_{p}')};")
            self.lines.extend(body)
            cur, lo = outs, lo_out
        return cur, lo

    def exchange(self, cur: list[str], lo: int, ind: str, tag: str = "") -> list[str]:
        """Shared-memory transpose from partition `lo` to the top-bit partition.
        Layout per window: lane group g = s >> top at offset g*G, G = 2^top + 32/T
        words, window stride XS = T*G + 4: the row reads (LDS.128) and the
        body-exchange scalar writes are bank-conflict-free."""
        top = self.k - self.tau
        G = self.G
        assert lo + self.tau <= top
        self.emit(f"{ind}// exchange: partition [{lo},{lo + self.tau}) -> [{top},{top + self.tau})")
        self.emit(f"{ind}__syncwarp(gmask);")
        lowmask = (1 << top) - 1
        r = 0
        while r < self.SL:
            s0 = self.state_of(r, 0, lo)
            run = 1
            while r + run < self.SL and self.state_of(r + run, 0, lo) == s0 + run and run < 4:
                run += 1
            off = (s0 & lowmask) + G * (s0 >> top)
            if run == 4 and off % 4 == 0:
                self.emit(f"{ind}*reinterpret_cast<int4*>(xw + {off} + (t << {lo})) = "
                          f"make_int4({cur[r]}, {cur[r + 1]}, {cur[r + 2]}, {cur[r + 3]});")
                r += 4
            else:
                self.emit(f"{ind}xw[{off} + (t << {lo})] = {cur[r]};")
                r += 1
        self.emit(f"{ind}__syncwarp(gmask);")
        out = []
        for r in range(0, self.SL, 4):
            nm = f"yx{tag}_{r}"
            self.emit(f"{ind}const int4 {nm} = *reinterpret_cast<const int4*>(xr + {r});")
            out += [f"{nm}.x", f"{nm}.y", f"{nm}.z", f"{nm}.w"]
        return out

    def shift_cur(self, ind: str) -> None:
        """cur <- cur advanced by P*B bytes (the next body's stages)."""
        nb = self.P * self.B
        qw, rb = nb // 4, nb % 4
        for i in range(self.NWC):
            a = f"cur[{i + qw}]" if i + qw < self.NWC else "0u"
            if rb == 0:
                self.emit(f"{ind}cur[{i}] = {a};")
            else:
                b = f"cur[{i + qw + 1}]" if i + qw + 1 < self.NWC else "0u"
                self.emit(f"{ind}cur[{i}] = __funnelshift_r({a}, {b}, {8 * rb});")

    # -- whole kernel ----------------------------------------------------------
    def kernel(self) -> str:
        K, B, S, SL, T, tau = self.K, self.B, self.S, self.SL, self.T, self.tau
        BL, NL, NWC, SQ, P, NIT, R = self.BL, self.NL, self.NWC, self.SQ, self.P, self.NIT, self.R
        WPC = NT // T
        xstride = self.XS
        top = self.top
        lo_end = top - R if tau else 0  # lane partition of the metrics at block end
        self.lo_end = lo_end
        name = f"vtk_{self.name}"
        e = self.emit
        e("// GENERATED by gen_kernels.py -- do not edit.")
        e(f"// code {self.name}: K={K}, generators (octal) {', '.join(oct(g)[2:] for g in self.gens)}; "
          f"{T} lane(s)/window, {SL} metrics/lane; history block = {NIT} x {P}-stage loop body + {R}-stage tail")
        e('#include "../vt_common.cuh"')
        e("")
        e(f'extern "C" __global__ void __launch_bounds__({NT}, 1) {name}(const vt::StreamArgs a) {{')
        e(f"  constexpr int B = {B}, K = {K}, BL = {BL}, NL = {NL}, NWC = {NWC};")
        e("  const int tid = threadIdx.x;")
        e(f"  const int t = tid & {T - 1};")
        e(f"  const int wloc = tid >> {tau};")
        if self.dyn_smem:  # over the 48 KB static limit (e.g. K=8 with three outputs): dynamic
            e("  extern __shared__ __align__(16) uint4 smem_dyn[];")
            e("  uint4* const s_llr = smem_dyn;")
            e(f"  uint32_t* const s_tb = reinterpret_cast<uint32_t*>(smem_dyn + NL * {NT});")
            if T > 1:
                e(f"  int32_t* const xs = reinterpret_cast<int32_t*>(s_tb + {NT});")
        else:
            e(f"  __shared__ __align__(16) uint4 s_llr[NL * {NT}];")
            e(f"  __shared__ uint32_t s_tb[{NT}];")
        if T > 1:
            if not self.dyn_smem:
                e(f"  __shared__ __align__(16) int32_t xs[{WPC} * {xstride}];")
            e(f"  int32_t* const xw = xs + wloc * {xstride};")
            e(f"  const int32_t* const xr = xw + t * {self.G};")
            e("  const int lane0 = (tid & 31) & ~%d;" % (T - 1))
            e(f"  const unsigned gmask = {(1 << T) - 1}u << lane0;  // this window's lanes (bodies may diverge per window)")
            for n in range(P):
                lo_in = top - n
                for b, g in enumerate(self.gens):
                    e(f"  const int32_t f{n}_{b} = 1 - 2 * (__popc({g}u & ((unsigned)t << {lo_in})) & 1);")
        e("  const uint64_t pol_first = vt::policy_evict_first();")
        e("  const uint64_t pol_last = vt::policy_evict_last();")
        e("  const int64_t nwin = a.w1 - a.w0;")
        e("  const int64_t buf_bytes = (a.st1 - a.st0) * B;")
        e(f"  uint4* const slot = a.scratch + (size_t)blockIdx.x * a.nbs * {SQ} * {NT} + tid;")
        e("  uint4* const wslot = slot - t;  // lane 0 of this window's lane group")
        e("  uint4* const my_llr = s_llr + tid;")
        e("  vt::Traceback<K, BL> tb;")
        e("  tb.running = false;")
        e("  tb.active = false;")
        e("  int parity_prev = 0, parity = 0;")
        # (lane, slot) of state j at block end, and the address of its history word
        if tau:
            tl_expr = f"(j >> {lo_end}) & {T - 1}"
            r_expr = f"((j >> {lo_end + tau}) << {lo_end}) | (j & {(1 << lo_end) - 1})"
        else:
            tl_expr, r_expr = "0", "j"
        e("  auto field_word = [&](int blk, uint32_t j, int par, uint32_t& half) -> const uint32_t* {")
        e("    const int bs = blk - a.b_lo;")
        e("    const int x = par ? (a.nbs - 1 - bs) : bs;")
        e(f"    const uint32_t tl = {tl_expr}, r = {r_expr};")
        e("    half = r & 1;")
        e(f"    const uint4* q = wslot + tl + ((size_t)x * {SQ} + (r >> 3)) * {NT};")
        e("    return reinterpret_cast<const uint32_t*>(q) + ((r & 7) >> 1);")
        e("  };")
        e(f"  for (int64_t tile = blockIdx.x; tile * {WPC} < nwin; tile += gridDim.x, parity ^= 1) {{")
        e(f"    const int64_t wrel = tile * {WPC} + wloc;")
        e("    // the previous tile's history stores (read back by this tile's traceback steps with")
        e("    // cp.async, by lane 0 of the window's lanes) are ordered before those reads")
        e("    __threadfence();")
        if T > 1:
            e("    __syncwarp(gmask);")
        e("    const bool active = wrel < nwin;")
        e("    const vt::Window g = vt::window_geometry<BL>(a, a.w0 + (active ? wrel : nwin - 1));")
        e("    const int64_t o0 = (g.g0 - a.st0) * B;")
        e("    " + " ".join(f"int32_t m{r} = 0;" for r in range(SL)))
        e("    int32_t rfold = 0;")
        e("    int64_t offset = 0;")
        e("    uint32_t cur[NWC];")
        e("    // leading zero-LLR padding keeps all-zero metrics at zero: skip whole loop bodies of it")
        e(f"    int it_start = (int)min(max(g.s - g.g0, (int64_t)0) / {P}, (int64_t){NIT});")
        e(f"    const int64_t o0s = o0 + (int64_t)it_start * {P * B};")
        e("    vt::stage_llr<NL, %d>(my_llr, a.llr, buf_bytes, o0s, pol_first);" % NT)
        e("    vt::cp_async_wait_all();")
        e("    vt::realign<NL, NWC, %d>(cur, my_llr, (int)(o0s & 15), "
          f"(int)min(max((g.s - g.g0 - (int64_t)it_start * {P}) * B, (int64_t)0), (int64_t)BL * B));" % NT)
        e("    for (int c = 0; c < a.nc; ++c) {")
        e("      const int64_t on = o0 + (int64_t)BL * B * (c + 1);")
        e("      if (c + 1 < a.nc) vt::stage_llr<NL, %d>(my_llr, a.llr, buf_bytes, on, pol_first);" % NT)
        e("      // one traceback step of the previous tile; the field load overlaps this chunk's ACS")
        e("      const bool tb_load = (t == 0) && tb.running && tb.b >= a.b_lo;")
        e("      uint32_t tb_half = 0;")
        e("      if (tb_load) vt::cp_async4(&s_tb[tid], field_word(tb.b, tb.j, parity_prev, tb_half));")
        e("      // history codes only in blocks whose decisions are stored (warm-up blocks need none)")
        e("      const int32_t cflag = (c >= a.b_lo) ? 1 : 0;")
        e(f"      int32_t cmul = cflag << ({P} * it_start);")
        e("#pragma unroll 1")
        e(f"      for (int it = it_start; it < {NIT}; ++it) {{")
        names, lo = self.body("        ", P, [f"m{r}" for r in range(SL)], top, "",
                              lambda q, d: f"vt::mad_fma(cmul, {1 << q}, {d})")
        if T > 1:
            names = self.exchange(names, lo, "        ", tag="b")
        for r in range(SL):
            e(f"        m{r} = {names[r]};")
        self.shift_cur("        ")
        e(f"        cmul <<= {P};")
        e("        rfold = 0;")
        e("      }")
        e("      it_start = 0;")
        fin = [f"m{r}" for r in range(SL)]
        if R:
            fin, lo = self.body("      ", R, fin, top, "t",
                                lambda q, d: f"vt::mad_fma(cflag, {1 << (P * NIT + q)}, {d})")
            assert lo == lo_end
        e("      rfold = 0;")
        e("      vt::cp_async_wait_all();")
        e("      if (tb_load) tb.step(a, (s_tb[tid] >> (16 * tb_half)) & 0xFFFFu);")
        # block end: histories to scratch, clear
        e("      if (c >= a.b_lo) {")
        e("        const int bs = c - a.b_lo;")
        e(f"        uint4* const dst = slot + (size_t)(parity ? (a.nbs - 1 - bs) : bs) * {SQ} * {NT};")
        for gq in range(0, SL, 8):
            w = []
            for h in range(4):
                ra, rb = gq + 2 * h, gq + 2 * h + 1
                a_ = fin[ra] if ra < SL else "0"
                b_ = fin[rb] if rb < SL else "0"
                w.append(f"vt::prmt((uint32_t){a_}, (uint32_t){b_}, 0x5410u)")
            e(f"        vt::st_global_v4_hint(dst + {gq // 8} * {NT}, make_uint4({', '.join(w)}), pol_last);")
        e("      }")
        for r in range(SL):
            e(f"      const int32_t z{r} = {fin[r]} & (int32_t)0xFFFF0000;")
        if T > 1:
            e("      rfold = __shfl_sync(0xFFFFFFFFu, z0, lane0);")
        else:
            e("      rfold = z0;")
        e("      if (c + 1 < a.nc) {")
        if T > 1:
            nxt = self.exchange([f"z{r}" for r in range(SL)], lo_end, "        ", tag="e")
        else:
            nxt = [f"z{r}" for r in range(SL)]
        for r in range(SL):
            e(f"        m{r} = {nxt[r]};")
        e("        offset += (rfold >> 16);")
        e("        vt::realign<NL, NWC, %d>(cur, my_llr, (int)(on & 15), "
          "(int)min(max((g.s - (g.g0 + (int64_t)BL * (c + 1))) * B, (int64_t)0), (int64_t)BL * B));" % NT)
        e("      } else {")
        for r in range(SL):
            e(f"        m{r} = z{r};")
        e("      }")
        e("    }")
        e("    if (t == 0 && tb.running) tb.drain_unstored(a);")
        # argmax in the block-end partition: key = M | (S-1-j)
        e("    // final state: argmax, lowest index on ties (reference.py:138)")
        tsh = f"(t << {lo_end})" if tau else "0"
        keys = [f"(m{r} | ({S - 1 - self.state_of(r, 0, lo_end)} - {tsh}))" for r in range(SL)]
        e(f"    int32_t best = {keys[0]};")
        for r in range(1, SL):
            e(f"    best = max(best, {keys[r]});")
        for d in range(tau):
            e(f"    best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, {1 << d}));")
        e(f"    const uint32_t jst = (uint32_t)({S - 1} - (best & 0xFFFF));")
        e("    if (t == 0 && active && a.final_metric) a.final_metric[wrel] = (int64_t)(best >> 16) + offset;")
        e("    if (t == 0) tb.start(g, jst, active, a.nc, a.N);")
        e("    parity_prev = parity;")
        e("  }")
        e("  // traceback of the CTA's last tile (no following tile to hide it behind)")
        e("  if (t == 0) {")
        e("    while (tb.running && tb.b >= a.b_lo) {")
        e("      uint32_t half;")
        e("      const uint32_t w = *field_word(tb.b, tb.j, parity_prev, half);")
        e("      tb.step(a, (w >> (16 * half)) & 0xFFFFu);")
        e("    }")
        e("    if (tb.running) tb.drain_unstored(a);")
        e("  }")
        e("}")
        e("")
        return "\n".join(self.lines)


def _gen16_supported(name: str, K: int, gens: tuple[int, ...]) -> bool:
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    from gen_kernels16 import Gen16
    return Gen16(name, K, gens).supported


REGISTRY_HEADER = [
    "// GENERATED by gen_kernels.py -- kernel registry:",
    "// VT_KERNEL(fn, fn without final metrics or nullptr, dynamic smem bytes, tensor-core BM, threads per CTA, K, B, "
    "lanes/window T, windows/thread, SL, chunk CH, history group BL, uint4/group SQ, body stages, TMA row lines, {gens})",
    "",
]


def code_units(name: str, K: int, gens: tuple[int, ...]) -> list[tuple[str, str, list[str], list[str]]]:
    """Every kernel form generated for one code: (file name, CUDA source, declarations,
    registry lines).  Used by the build (STANDARD_CODES) and by the runtime code JIT
    (paper_2011_13579_b200/jit.py), so both produce the same kernels."""
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    if here not in sys.path:
        sys.path.insert(0, here)
    units = []
    gl = ", ".join(f"{x}u" for x in gens)
    T = threads_per_window(K)
    g = Gen(name, K, gens, T)
    units.append((f"vtk_{name}.cu", g.kernel(),
                  [f'extern "C" __global__ void vtk_{name}(const vt::StreamArgs a);'],
                  [f"VT_KERNEL(vtk_{name}, nullptr, {g.SMEM_DYN}, 0, {NT}, {K}, {len(gens)}, {T}, 1, {g.SL}, {g.BL}, {g.BL}, "
                   f"{g.SQ}, 0, 0, {{{gl}}})"]))
    lanes = T if K in (8, 9) else 0  # (K=7 over 2 lanes measured 97.6 vs 165 Gbps: DESIGN §9b)
    if lanes:  # packed 16x2 variant over T lanes per window pair
        from gen_kernels16m import Gen16M
        gm = Gen16M(name, K, gens, lanes)
        # the host's padding-skip hazard check (vt_capi.cu launch_grid) uses the body length
        assert gm.CH % gm.P == 0 and gm.P % gm.L == 0
    if lanes and gm.supported:  # (the s32 kernels alone when the 16-bit range does not fit)
        units.append((f"vtk16m_{name}.cu", gm.kernel(),
                      [f'extern "C" __global__ void vtk16m_{name}(const vt::StreamArgs a);',
                       f'extern "C" __global__ void vtk16mnf_{name}(const vt::StreamArgs a);'],
                      [f"VT_KERNEL(vtk16m_{name}, &vtk16mnf_{name}, {gm.SMEM}, 0, 128, {K}, {len(gens)}, {lanes}, 2, "
                       f"{gm.SL}, {gm.CH}, {gm.L}, {gm.SQ}, {gm.P}, 0, {{{gl}}})"]))
    if K == 7 and _gen16_supported(name, K, gens):  # packed 16x2 variant: two windows per thread
        import gen_kernels16
        from gen_kernels16 import Gen16
        g16 = Gen16(name, K, gens)
        if g16.cheap and g16.B == 2 and gen_kernels16.NT == 128:  # tensor-core branch-metric variant (VT_KERNEL_VARIANT=16x2tc)
            gtc = Gen16(name, K, gens, tc=True)
            units.append((f"vtk16tc_{name}.cu", gtc.kernel(),
                          [f'extern "C" __global__ void vtk16tc_{name}(const vt::StreamArgs a);',
                           f'extern "C" __global__ void vtk16tcnf_{name}(const vt::StreamArgs a);'],
                          [f"VT_KERNEL(vtk16tc_{name}, &vtk16tcnf_{name}, {gtc.SMEM}, 1, 128, {K}, {len(gens)}, 1, 2, "
                           f"{gtc.S}, {gtc.CH}, {gtc.L}, {gtc.S // 16}, {gtc.P}, 0, {{{gl}}})"]))
        targ = ", const __grid_constant__ CUtensorMap tmap" if g16.tma else ""
        rows = g16.RS if g16.tma else 0  # TMA box lines per row (0: no tensor-map parameter)
        if g16.cheap and g16.B == 2 and gen_kernels16.NT == 128:  # mma.sync branch metrics (VT_KERNEL_VARIANT=16x2mma)
            gmx = Gen16(name, K, gens, mma=True)
            units.append((f"vtk16mma_{name}.cu", gmx.kernel(),
                          [f'extern "C" __global__ void vtk16mma_{name}(const vt::StreamArgs a{targ});',
                           f'extern "C" __global__ void vtk16mmanf_{name}(const vt::StreamArgs a{targ});'],
                          [f"VT_KERNEL(vtk16mma_{name}, &vtk16mmanf_{name}, {gmx.SMEM}, 2, 128, {K}, {len(gens)}, 1, 2, "
                           f"{gmx.S}, {gmx.CH}, {gmx.L}, {gmx.S // 16}, {gmx.P}, {rows}, {{{gl}}})"]))
        units.append((f"vtk16_{name}.cu", g16.kernel(),
                      [f'extern "C" __global__ void vtk16_{name}(const vt::StreamArgs a{targ});',
                       f'extern "C" __global__ void vtk16nf_{name}(const vt::StreamArgs a{targ});'],
                      [f"VT_KERNEL(vtk16_{name}, &vtk16nf_{name}, {g16.SMEM}, {3 if g16.tmh else 0}, {gen_kernels16.NT}, {K}, {len(gens)}, "
                       f"1, 2, {g16.S}, {g16.CH}, {g16.L}, {g16.S // 16}, {g16.P}, {rows}, {{{gl}}})"]))
    return units


def _write_if_changed(path: str, text: str) -> None:
    if not os.path.exists(path) or open(path).read() != text:
        with open(path, "w") as fh:
            fh.write(text)


def generate(outdir: str, codes: dict | None = None) -> list[str]:
    codes = codes or STANDARD_CODES
    os.makedirs(outdir, exist_ok=True)
    files = []
    reg = list(REGISTRY_HEADER)
    decl = ["// GENERATED by gen_kernels.py -- kernel declarations", '#include "../vt_common.cuh"', ""]
    for name, (K, polys) in codes.items():
        gens = tuple(int(p, 8) for p in polys)
        for fname, src, d, r in code_units(name, K, gens):
            path = os.path.join(outdir, fname)
            _write_if_changed(path, src)
            files.append(path)
            decl.extend(d)
            reg.extend(r)
    for fname, lines in (("registry.inc", reg), ("registry_decl.inc", decl)):
        _write_if_changed(os.path.join(outdir, fname), "\n".join(lines) + "\n")
    for stale in set(os.listdir(outdir)) - {os.path.basename(f) for f in files}:  # kernels no longer generated
        if stale.endswith(".cu"):
            os.remove(os.path.join(outdir, stale))
    return files


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "gen"))
    args = ap.parse_args()
    for f in generate(args.out):
        print(f)
