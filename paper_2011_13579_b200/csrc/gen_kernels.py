#!/usr/bin/env python3
"""Generate straight-line sm_100a ACS kernels, one per convolutional code.

Why a generator: the add-compare-select recursion for 2^(K-1) states over a
16-stage block is ~2,100 independent integer ops per thread.  Written as C++
loops over register arrays, NVVM needs minutes per kernel and spends ~2x the
registers; emitted as straight-line SSA code it compiles in about a second and
ptxas sees exactly the dataflow we want (IMAD.IADD on the FMA pipe feeding one
DPX VIADDMNMX on the ALU pipe per state-stage).

Reference semantics implemented (pkg/src/vitertile):
  * reference.py:60-83  predecessors i0 = 2*(j mod 2^(K-2)), i1 = i0+1, input u = j >> (K-2)
  * codes.py:183-193    branch output bit b = parity(g_b & ((u << (K-1)) | i))
  * reference.py:86-92,119-120  branch metric = sum_b (1 - 2*bit_b) * llr_b (maximised)
  * reference.py:121    tie -> second predecessor: the i1 candidate carries +2^p in the
                        history bits, so signed max picks it on equal metrics
  * reference.py:124-125 renormalisation (exact): -lambda_0 folded into the branch metrics
  * reference.py:138    final state = lowest-index argmax
  * framing.py:68-141   windows / emit ranges (vt_common.cuh)

Threads per window T: K <= 7 keeps all 2^(K-1) metrics in one thread (T=1).
K = 8, 9 spread them over T = 2, 4 lanes.  With the lanes partitioned by tau =
log2(T) state bits that start at the top, a radix-2 stage maps a partition at
bits [lo, lo+tau) onto [lo-1, lo-1+tau) with no data exchange, so K-1-tau stages
run exchange-free; then one shared-memory transpose restores the top-bit
partition.  The lane-dependent part of the branch parity is a per-lane LLR sign
flip, so all lanes execute identical code.
"""
from __future__ import annotations

import argparse
import os

STANDARD_CODES = {
    # name: (K, generators as octal strings)   -- BASELINE.json configs + tests/conftest.py:7-15
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
        assert self.SL % 8 == 0 or self.SL < 8, "slots per lane must pack into uint4 groups"
        self.period = (self.k - self.tau) if T > 1 else 10 ** 9
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

    # -- one 16-stage block ----------------------------------------------------
    def block(self, cur: list[str], lo: int) -> tuple[list[str], int, list[int]]:
        """Emit 16 stages starting from names `cur` in partition `lo`.
        Returns (names, partition at block end, exchange positions)."""
        B = self.B
        n_in_group = 0
        xchg = []
        for q in range(16):
            if self.T > 1 and n_in_group == self.period:
                cur = self.exchange(cur, lo, tag=f"q{q}")
                lo = self.k - self.tau
                n_in_group = 0
                xchg.append(q)
            lo_out = lo - 1 if self.tau else lo
            # LLRs of this stage (bytes q*B + b of the chunk), as llr << 16
            for b in range(B):
                byte = q * B + b
                expr = f"vt::llr_hi16(cur[{byte >> 2}], {byte & 3}u)"
                if self.T > 1:
                    expr = f"{expr} * f{n_in_group}_{b}"
                self.emit(f"      const int32_t L{q}_{b} = {expr};")
            outs = []
            body = []
            need_d, need_e = set(), set()
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
                nm = f"x{q}_{r}"
                body.append(f"      const int32_t {nm} = vt::addmax({cur[r0]}, D{q}_{p0}, "
                            f"vt::add_fma({cur[r1]}, E{q}_{p1}));")
                outs.append(nm)
            for p in sorted(need_d | need_e):
                terms = []
                for b in range(B):
                    sgn = "-" if (p >> b) & 1 else "+"
                    terms.append(f"{sgn} L{q}_{b}")
                expr = " ".join(terms).lstrip("+ ")
                if q == 0:
                    expr = f"{expr} - rfold"
                self.emit(f"      const int32_t D{q}_{p} = {expr};")
                if p in need_e:
                    self.emit(f"      const int32_t E{q}_{p} = D{q}_{p} + {1 << q};")
            self.lines.extend(body)
            cur = outs
            lo = lo_out
            n_in_group += 1
        return cur, lo, xchg

    def exchange(self, cur: list[str], lo: int, tag: str) -> list[str]:
        """Shared-memory transpose from partition `lo` to the top-bit partition."""
        top = self.k - self.tau
        self.emit(f"      // exchange ({tag}): partition [{lo},{lo + self.tau}) -> [{top},{top + self.tau})")
        self.emit("      __syncwarp();")
        r = 0
        while r < self.SL:
            s0 = self.state_of(r, 0, lo)
            run = 1
            while (r + run < self.SL and self.state_of(r + run, 0, lo) == s0 + run and run < 4):
                run += 1
            if run == 4 and s0 % 4 == 0:
                self.emit(f"      *reinterpret_cast<int4*>(xw + {s0} + (t << {lo})) = "
                          f"make_int4({cur[r]}, {cur[r + 1]}, {cur[r + 2]}, {cur[r + 3]});")
                r += 4
            else:
                self.emit(f"      xw[{s0} + (t << {lo})] = {cur[r]};")
                r += 1
        self.emit("      __syncwarp();")
        out = []
        for r in range(0, self.SL, 4):
            nm = f"y{tag}_{r}"
            self.emit(f"      const int4 {nm} = *reinterpret_cast<const int4*>(xr + {r});")
            out += [f"{nm}.x", f"{nm}.y", f"{nm}.z", f"{nm}.w"]
        return out

    # -- whole kernel ----------------------------------------------------------
    def kernel(self) -> str:
        K, B, S, SL, T, tau = self.K, self.B, self.S, self.SL, self.T, self.tau
        WPC = NT // T
        xstride = S + (4 if T > 1 else 0)
        name = f"vtk_{self.name}"
        e = self.emit
        e("// GENERATED by gen_kernels.py -- do not edit.")
        e(f"// code {self.name}: K={K}, generators (octal) {', '.join(oct(g)[2:] for g in self.gens)}, "
          f"{T} lane(s) per window, {SL} metrics per lane")
        e('#include "../vt_common.cuh"')
        e("")
        e(f'extern "C" __global__ void __launch_bounds__({NT}, 1) {name}(const vt::StreamArgs a) {{')
        e(f"  constexpr int B = {B};")
        e("  const int tid = threadIdx.x;")
        e(f"  const int t = tid & {T - 1};")
        e(f"  const int wloc = tid >> {tau};")
        if T > 1:
            e(f"  __shared__ __align__(16) int32_t xs[{WPC} * {xstride}];")
            e(f"  int32_t* const xw = xs + wloc * {xstride};")
            e(f"  const int32_t* const xr = xw + (t << {self.k - tau});")
            e("  const unsigned gmask = 0xFFFFFFFFu;")
            e(f"  const int lane0 = (tid & 31) & ~{T - 1};")
            # per-lane LLR sign flips for stage n of an exchange period
            for n in range(min(self.period, 16)):
                lo_in = self.k - tau - n
                for b, g in enumerate(self.gens):
                    e(f"  const int32_t f{n}_{b} = 1 - 2 * (__popc({g}u & ((unsigned)t << {lo_in})) & 1);")
        e("  const int64_t nwin = a.w1 - a.w0;")
        e("  const int64_t buf_bytes = (a.st1 - a.st0) * B;")
        e(f"  uint4* const slot = a.scratch + (size_t)blockIdx.x * a.nbs * {max(SL // 8, 1)} * {NT} + tid;")
        e(f"  for (int64_t tile = blockIdx.x; tile * {WPC} < nwin; tile += gridDim.x) {{")
        e(f"    const int64_t wrel = tile * {WPC} + wloc;")
        e("    const bool active = wrel < nwin;")
        e("    const vt::Window g = vt::window_geometry(a, a.w0 + (active ? wrel : nwin - 1));")
        e("    const int64_t o0 = (g.g0 - a.st0) * B;")
        e("    const int shift = (int)(o0 & 15);")
        top = self.k - tau if tau else 0
        e("    " + " ".join(f"int32_t m{r} = 0;" for r in range(SL)))
        e("    int32_t rfold = 0;")
        e("    int64_t offset = 0;")
        e("    uint4 raw[B + 1];")
        e("    uint32_t cur[4 * B];")
        e("    vt::load_raw<B>(raw, a.llr, buf_bytes, o0);")
        e("    vt::realign<B>(cur, raw, shift, (int)min(max((g.s - g.g0) * B, (int64_t)0), (int64_t)16 * B));")
        e("    for (int c = 0; c < a.nc; ++c) {")
        e("      if (c + 1 < a.nc) vt::load_raw<B>(raw, a.llr, buf_bytes, o0 + (int64_t)16 * B * (c + 1));")
        names, lo_end, xchg = self.block([f"m{r}" for r in range(SL)], top)
        self.lo_end = lo_end
        # block end: stream histories, clear them
        e("      if (c >= a.b_lo) {")
        e(f"        uint4* const dst = slot + (size_t)(c - a.b_lo) * {max(SL // 8, 1)} * {NT};")
        for gq in range(0, SL, 8):
            w = []
            for h in range(4):
                ra, rb = gq + 2 * h, gq + 2 * h + 1
                a_ = names[ra] if ra < SL else "0"
                b_ = names[rb] if rb < SL else "0"
                w.append(f"vt::prmt((uint32_t){a_}, (uint32_t){b_}, 0x5410u)")
            e(f"        dst[{gq // 8} * {NT}] = make_uint4({', '.join(w)});")
        if SL < 8:  # small codes: pad the single uint4 group
            pass
        e("      }")
        for r in range(SL):
            e(f"      const int32_t z{r} = {names[r]} & (int32_t)0xFFFF0000;")
        if T > 1:
            e("      rfold = __shfl_sync(gmask, z0, lane0);")
        else:
            e("      rfold = z0;")
        e("      if (c + 1 < a.nc) {")
        if T > 1:
            nxt = self.exchange([f"z{r}" for r in range(SL)], lo_end, tag="blk")
            for r in range(SL):
                e(f"        m{r} = {nxt[r]};")
        else:
            for r in range(SL):
                e(f"        m{r} = z{r};")
        e("        offset += (rfold >> 16);")
        e("        vt::realign<B>(cur, raw, shift, "
          "(int)min(max((g.s - (g.g0 + 16 * (int64_t)(c + 1))) * B, (int64_t)0), (int64_t)16 * B));")
        e("      } else {")
        for r in range(SL):
            e(f"        m{r} = z{r};")
        e("      }")
        e("    }")
        # argmax (lowest index on ties): key = M | (S-1-j)
        e(f"    // final state: argmax, lowest index on ties (reference.py:138); partition [{lo_end},{lo_end + tau})")
        tsh = f"(t << {lo_end})" if tau else "0"
        keys = []
        for r in range(SL):
            j0 = self.state_of(r, 0, lo_end)
            keys.append(f"(m{r} | ({S - 1 - j0} - {tsh}))")
        e(f"    int32_t best = {keys[0]};")
        for r in range(1, SL):
            e(f"    best = max(best, {keys[r]});")
        if T > 1:
            for d in range(tau):
                e(f"    best = max(best, __shfl_xor_sync(gmask, best, {1 << d}));")
        e(f"    const uint32_t jst = (uint32_t)({S - 1} - (best & 0xFFFF));")
        e(f"    if (t == 0 && active && a.final_metric) a.final_metric[wrel] = (int64_t)(best >> 16) + offset;")
        # traceback (one lane per window)
        e("    if (t == 0) {")
        e(f"      uint4* const wslot = slot - t;  // lane 0 of this window")
        e("      vt::traceback_emit<%d>(a, g, jst, active, [&](int bs, uint32_t j) -> uint32_t {" % K)
        if tau:
            e(f"        const uint32_t tl = (j >> {lo_end}) & {T - 1};")
            e(f"        const uint32_t r = ((j >> {lo_end + tau}) << {lo_end}) | (j & {(1 << lo_end) - 1});")
        else:
            e("        const uint32_t tl = 0, r = j;")
        e(f"        const uint4* q = wslot + tl + ((size_t)bs * {max(SL // 8, 1)} + (r >> 3)) * {NT};")
        e("        return (uint32_t)reinterpret_cast<const uint16_t*>(q)[r & 7];")
        e("      });")
        e("    }")
        e("  }")
        e("}")
        e("")
        return "\n".join(self.lines)


def generate(outdir: str, codes: dict | None = None) -> list[str]:
    codes = codes or STANDARD_CODES
    os.makedirs(outdir, exist_ok=True)
    files = []
    reg = ["// GENERATED by gen_kernels.py -- kernel registry", ""]
    decl = ["// GENERATED by gen_kernels.py -- kernel declarations", '#include "../vt_common.cuh"', ""]
    for name, (K, polys) in codes.items():
        gens = tuple(int(p, 8) for p in polys)
        T = threads_per_window(K)
        g = Gen(name, K, gens, T)
        src = g.kernel()
        path = os.path.join(outdir, f"vtk_{name}.cu")
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as fh:
                fh.write(src)
        files.append(path)
        gl = ", ".join(f"{x}u" for x in gens)
        decl.append(f'extern "C" __global__ void vtk_{name}(const vt::StreamArgs a);')
        reg.append(f"VT_KERNEL(vtk_{name}, {K}, {len(gens)}, {T}, {g.SL}, {{{gl}}})")
    for fname, lines in (("registry.inc", reg), ("registry_decl.inc", decl)):
        rpath = os.path.join(outdir, fname)
        text = "\n".join(lines) + "\n"
        if not os.path.exists(rpath) or open(rpath).read() != text:
            with open(rpath, "w") as fh:
                fh.write(text)
    return files


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "gen"))
    args = ap.parse_args()
    for f in generate(args.out):
        print(f)
