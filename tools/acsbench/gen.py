#!/usr/bin/env python3
"""ACS-rate microbenchmark generator (design exploration, not product code).

Emits acs_bench.cu with K=7 (171,133) ACS loop kernels that mimic the decoder's
inner loop without framing/traceback, to measure achievable state-updates per
cycle per SM on the B200 for different instruction forms and group-end schemes:
  v16     : 16x2 packed, VIADD.16x2 + VIADDMNMX.U16x2, no history extraction
  v16imad : 16x2 packed, carry-free 32-bit IMAD + VIADDMNMX.U16x2
  v16g    : v16 + L=3 group end (mask, pack, clear, st.global)
  v16gi   : v16imad + group end
  s32     : s32 IMAD + VIADDMNMX (one window per thread)
LLR bytes come from a per-thread shared-memory column (like the decoder).
"""
import sys

K = 7
S = 64
GENS = (0o171, 0o133)


def parity(x):
    return bin(x).count("1") & 1


def pattern(i, u):
    reg = (u << 6) | i
    return sum(parity(g & reg) << b for b, g in enumerate(GENS))


def gen_kernel(name, mode, L=3):
    imad = "imad" in mode or mode.endswith("i")
    group = mode.startswith("v16g")
    s32 = mode == "s32"
    o = []
    e = o.append
    e(f'extern "C" __global__ void __launch_bounds__(128, 1) {name}(const uint32_t* __restrict__ llrsrc, uint4* __restrict__ scratch, uint32_t* out, int iters) {{')
    e("  __shared__ uint32_t s_llr[64 * 128];")
    e("  const int tid = threadIdx.x;")
    e("  for (int i = 0; i < 64; ++i) s_llr[i * 128 + tid] = llrsrc[(blockIdx.x * 64 + i) * 128 + tid];")
    e("  __syncwarp();")
    e("  uint4* slot = scratch + (size_t)blockIdx.x * 128 * 64 + tid;")
    e("  const uint64_t pol = vt::policy_evict_last();")
    e("  " + " ".join(f"uint32_t m{j} = {j}u;" for j in range(S)))
    e("  uint32_t negR = 0;")
    e("  int gidx = 0;")
    e("#pragma unroll 1")
    e("  for (int it = 0; it < iters; ++it) {")
    e("    const uint32_t w0 = s_llr[((it * 3) & 63) * 128 + tid], w1 = s_llr[((it * 3 + 1) & 63) * 128 + tid], w2 = s_llr[((it * 3 + 2) & 63) * 128 + tid];")
    e("    const uint32_t cw[3] = {w0, w1, w2};")
    names = [f"m{j}" for j in range(S)]
    for q in range(6):
        # llr pair for both windows: bytes (2q, 2q+1) of cw for A, use same rotated for B
        if s32:
            e(f"    const int32_t L0_{q} = vt::llr_hi16(cw[{(2*q)//4}], {(2*q)%4}u), L1_{q} = vt::llr_hi16(cw[{(2*q+1)//4}], {(2*q+1)%4}u);")
            pats = {}
            for p in range(4):
                s0 = -1 if p & 1 else 1
                s1 = -1 if p & 2 else 1
                e(f"    const int32_t D{q}_{p} = {'' if s0 > 0 else '-'}L0_{q} {'+' if s1 > 0 else '-'} L1_{q};")
                e(f"    const int32_t E{q}_{p} = D{q}_{p} + {1 << (q % 6 + 4)};")
        else:
            gq = q % L
            e(f"    const uint32_t P{q}_0 = vt::prmt(cw[{(2*q)//4}], cw[{(2*q)//4}] ^ 0x5a5a5a5au, {((2*q)%4) | ((8 | ((2*q)%4)) << 4) | ((4 + (2*q)%4) << 8) | ((12 + (2*q)%4) << 12):#x}u);")
            e(f"    const uint32_t P{q}_1 = vt::prmt(cw[{(2*q+1)//4}], cw[{(2*q+1)//4}] ^ 0x5a5a5a5au, {((2*q+1)%4) | ((8 | ((2*q+1)%4)) << 4) | ((4 + (2*q+1)%4) << 8) | ((12 + (2*q+1)%4) << 12):#x}u);")
            for b in range(2):
                e(f"    const uint32_t U{q}_{b} = vt::vadd2(P{q}_{b}, 0x00800080u) << {L};")
                e(f"    const uint32_t N{q}_{b} = {(256 << L) * 0x10001:#x}u - U{q}_{b};")
            for p in range(4):
                expr = " + ".join(f"{'N' if (p >> b) & 1 else 'U'}{q}_{b}" for b in range(2))
                if gq == 0:
                    expr = f"vt::vadd2({expr}, negR)"
                e(f"    const uint32_t D{q}_{p} = {expr};")
                e(f"    const uint32_t E{q}_{p} = vt::vadd2(D{q}_{p}, {(1 << gq) * 0x10001:#x}u);")
        outs = []
        for j in range(S):
            u = j >> 5
            i0 = (j << 1) & 63
            i1 = i0 | 1
            p0, p1 = pattern(i0, u), pattern(i1, u)
            nm = f"x{q}_{j}"
            if s32:
                e(f"    const int32_t {nm} = vt::addmax((int32_t){names[i0]}, D{q}_{p0}, vt::add_fma((int32_t){names[i1]}, E{q}_{p1}));")
            elif imad:
                e(f"    const uint32_t {nm} = vt::vaddmax2({names[i0]}, D{q}_{p0}, vt::mad_u32({names[i1]}, 1u, E{q}_{p1}));")
            else:
                e(f"    const uint32_t {nm} = vt::vaddmax2({names[i0]}, D{q}_{p0}, vt::vadd2({names[i1]}, E{q}_{p1}));")
            outs.append(nm)
        names = outs
        if (not s32) and q % L == L - 1:
            for j in range(S):
                e(f"    m{j} = {names[j]};")
            names = [f"m{j}" for j in range(S)]
            lm = (0xFFFF & ~((1 << L) - 1)) * 0x10001
            e(f"    {{ const uint32_t r0 = m0 & {lm:#x}u; negR = vt::vadd2(~vt::vadd2(r0, 0xF400F400u), 0x00010001u); }}")
            if group and "gp" in mode:
                e("    {")
                e(f"      uint4* const dst = slot + (size_t)(gidx & 63) * 4 * 128;")
                ws = []
                for w in range(16):
                    a, b, c, d = 4 * w, 4 * w + 1, 4 * w + 2, 4 * w + 3
                    e(f"      const uint32_t p{w}a = vt::prmt(m{a}, m{b}, 0x6420u) & 0x07070707u;")
                    e(f"      const uint32_t p{w}b = vt::prmt(m{c}, m{d}, 0x6420u) & 0x07070707u;")
                    ws.append(f"vt::mad_u32(p{w}b, 8u, p{w}a)")
                for g in range(4):
                    e(f"      vt::st_global_v4_hint(dst + {g * 128}, make_uint4({', '.join(ws[4*g:4*g+4])}), pol);")
                if "nc" not in mode:
                    for j in range(S):
                        e(f"      m{j} &= 0xFFF8FFF8u;")
                e("    }")
                e("    ++gidx;")
            elif group:
                hm = ((1 << L) - 1) * 0x10001
                e("    {")
                e(f"      uint4* const dst = slot + (size_t)(gidx & 63) * 4 * 128;")
                for j in range(S):
                    e(f"      const uint32_t h{j} = m{j} & {hm:#x}u;")
                words = []
                for w in range(16):
                    acc = f"h{4 * w}"
                    for t in range(1, 4):
                        acc = f"vt::mad_u32(h{4 * w + t}, {1 << (L * t)}u, {acc})"
                    words.append(acc)
                for g in range(4):
                    e(f"      vt::st_global_v4_hint(dst + {g * 128}, make_uint4({', '.join(words[4*g:4*g+4])}), pol);")
                for j in range(S):
                    e(f"      m{j} = vt::mad_u32(h{j}, 0xFFFFFFFFu, m{j});")
                e("    }")
                e("    ++gidx;")
    for j in range(S):
        e(f"    m{j} = {names[j]};")
    if s32:
        e("    { const int32_t r = (int32_t)m0; " + " ".join(f"m{j} -= r;" for j in range(S)) + " }" if False else "")
    e("  }")
    e("  uint32_t acc = 0;")
    e("  " + " ".join(f"acc ^= m{j};" for j in range(S)))
    e("  out[blockIdx.x * 128 + tid] = acc;")
    e("}")
    return "\n".join(o)


MODES = ["v16", "v16imad", "v16g", "v16gi", "s32", "v16gpi", "v16gpnci"]
if __name__ == "__main__":
    out = ['#include "../../paper_2011_13579_b200/csrc/vt_common.cuh"', ""]
    for m in MODES:
        out.append(gen_kernel(f"acs_{m}", m))
    open(sys.argv[1], "w").write("\n".join(out))
