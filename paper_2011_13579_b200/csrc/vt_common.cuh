// Shared device helpers for the generated Viterbi kernels (gen_kernels.py).
//
// The generated kernels replace, per CUDA launch, the reference hot path
//   framing.decode_stream -> _decode_windows -> reference.decode_batch
//   (pkg/src/vitertile/framing.py:86-141, reference.py:95-144, 194-206).
// Everything here is the code that does not depend on the trellis: window
// geometry (framing.py:68-83), LLR chunk staging, survivor-history scratch
// addressing and the traceback / packed-bit emission.
#pragma once
#include <cstdint>
#include <cuda.h>  // (CUtensorMap only: the map is encoded on the host, vt_capi.cu)
#include <cuda_runtime.h>

namespace vt {

struct StreamArgs {
  const int8_t* llr;      // device buffer holding stages [st0, st1), layout (stage, B), 16-B aligned
  int64_t st0, st1;       // stage range held in llr (st0 multiple of 16, or 0)
  int64_t N;              // total stream length (stages)
  int64_t F, V;           // frame (payload) length and overlap (framing.py:68-83)
  int64_t w0, w1;         // window range decoded by this launch
  uint32_t* bits;         // packed output bits of the whole stream (LSB = earliest, cli.py:5-6)
  int64_t* final_metric;  // optional, per window (index w - w0): max path metric (reference.py:206)
  uint4* scratch;         // survivor-history scratch: gridDim.x * nbs * (S/T/8) * NT uint4
  int nc;                 // BL-stage chunks per window (uniform for the launch; BL = kernel block length)
  int b_lo;               // first chunk whose histories are stored
  int nbs;                // stored chunks per window (nc - b_lo)
  int tma;                // 1: the kernel's tensor-map parameter is valid (16x2 kernels stage LLR
                          // chunk rows with TMA): 3-D map over llr {16 bytes, 16-byte lines, 32 rows
                          // 2*F*B bytes apart} -- one box is the chunk rows of a warp's 32
                          // same-parity windows (interior windows are F*B bytes apart)
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}

// a + b issued on the FMA pipe (ptxas emits IMAD.IADD for mad a*1+b)
__device__ __forceinline__ int32_t add_fma(int32_t a, int32_t b) {
  int32_t d;
  asm("mad.lo.s32 %0, %1, 1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// a * b + c on the FMA pipe
__device__ __forceinline__ int32_t mad_fma(int32_t a, int32_t b, int32_t c) {
  int32_t d;
  asm("mad.lo.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// packed 16x2 ops (per-half modular add; unsigned max): VIADD.16x2 / VIADDMNMX.U16x2
__device__ __forceinline__ uint32_t vadd2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
// per-half unsigned min (ptxas fuses pairs into VIMNMX3.U16x2)
__device__ __forceinline__ uint32_t vmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("min.u16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t vaddmax2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("{.reg .b32 t; add.u16x2 t, %1, %2; max.u16x2 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
__device__ __forceinline__ uint32_t mad_u32(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// max(a + b, c): ptxas fuses add.s32 + max.s32 into one DPX VIADDMNMX (ALU pipe)
__device__ __forceinline__ int32_t addmax(int32_t a, int32_t b, int32_t c) {
  int32_t d;
  asm("{.reg .s32 t; add.s32 t, %1, %2; max.s32 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// --- asynchronous copies (cannot be sunk by the scheduler, unlike plain loads) ---
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// evict_last for the fraction FRAC of the accessed lines, evict_first for the rest
#define VT_POLICY_LAST_FIRST(FRAC)                                                                      \
  ([] {                                                                                                 \
    uint64_t p;                                                                                         \
    asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, " #FRAC ";" : "=l"(p)); \
    return p;                                                                                           \
  }())
// 16-byte global->shared copy; src_bytes = 0 zero-fills (out-of-range words).
// (No .L2::cache_hint operand: ptxas 12.9 allocated its 64-bit policy descriptor to
// an odd uniform register in the K=9 kernels, which traps as an illegal instruction.)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes, uint64_t /*pol*/) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// wait until at most N committed groups of this thread are still in flight
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void st_global_v4_hint(uint4* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// --- TMA (cp.async.bulk.tensor) + mbarrier completion (the 16x2 kernels' LLR staging) ---
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  do {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                 : "=r"(done) : "r"(b), "r"(parity) : "memory");
  } while (!done);
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// box {16, lines, rows} at coordinates (0, line, row) -> dst (rows of lines*16 bytes), completes on bar
__device__ __forceinline__ void tma_load_rows(void* dst, const CUtensorMap* map, int line, int row, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
      ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(map), "r"(0), "r"(line), "r"(row),
      "r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}

// Window geometry of window w (framing.py:78-82) in the end-aligned chunk frame.
struct Window {
  int64_t e0, e1;   // emit range
  int64_t s, stop;  // window range
  int64_t g0;       // stream stage of chunk 0 (= stop - BL*nc; may be < s: zero padding)
};

template <int BL>
__device__ __forceinline__ Window window_geometry(const StreamArgs& a, int64_t w) {
  Window g;
  g.e0 = w * a.F;
  g.e1 = min(g.e0 + a.F, a.N);
  g.s = max((int64_t)0, g.e0 - a.V);
  g.stop = min(a.N, g.e1 + a.V);
  g.g0 = g.stop - BL * (int64_t)a.nc;
  return g;
}

// Stage the 16-byte words covering LLR bytes [o, o + nb) of the buffer into
// this thread's shared slot (column layout smem[i * NT + tid]); words outside
// the buffer are zero-filled.  Completes at cp_async_wait_all().
template <int NL, int NT>
__device__ __forceinline__ void stage_llr(uint4* smem_col, const int8_t* __restrict__ llr, int64_t buf_bytes,
                                          int64_t o, uint64_t pol) {
  const int64_t base = (o >> 4) << 4;  // floor to 16 (arithmetic shift)
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    const int64_t a = base + 16 * i;
    const bool ok = (a >= 0) && (a < buf_bytes);
    cp_async16(smem_col + i * NT, llr + (ok ? a : 0), ok ? 16 : 0, pol);
  }
}

// Realign the staged words by the byte misalignment (o & 15) into NWC words
// holding bytes [o, o + 4*NWC); zero the first `zb` bytes (stages before the window).
template <int NL, int NWC, int NT>
__device__ __forceinline__ void realign(uint32_t (&out)[NWC], const uint4* smem_col, int shift, int zb) {
  constexpr int NW = 4 * NL;
  static_assert(NWC + 4 <= NW, "staging window too small");
  uint32_t w[NW];
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    const uint4 v = smem_col[i * NT];
    w[4 * i + 0] = v.x;
    w[4 * i + 1] = v.y;
    w[4 * i + 2] = v.z;
    w[4 * i + 3] = v.w;
  }
  const int q = shift >> 2, r = (shift & 3) * 8;
#pragma unroll
  for (int i = 0; i + 1 < NW; ++i) w[i] = (q & 1) ? w[i + 1] : w[i];
#pragma unroll
  for (int i = 0; i + 2 < NW; ++i) w[i] = (q & 2) ? w[i + 2] : w[i];
#pragma unroll
  for (int k = 0; k < NWC; ++k) out[k] = __funnelshift_r(w[k], w[k + 1], r);
  if (zb > 0) {
#pragma unroll
    for (int k = 0; k < NWC; ++k) {
      const int lo = zb - 4 * k;
      if (lo >= 4) out[k] = 0u;
      else if (lo > 0) out[k] &= 0xFFFFFFFFu << (8 * lo);
    }
  }
}

// Row-layout staging (16x2 kernels): each thread's NL staged 16-byte words are one
// contiguous 16*NL-byte row (row stride 48 B for NL=3: the 16-byte cp.async writes of
// 8 consecutive threads hit distinct banks).  `fast` = the whole span is inside the
// buffer (no per-word bounds checks).
template <int NL>
__device__ __forceinline__ void stage_row(char* row, const int8_t* __restrict__ llr, int64_t buf_bytes, int64_t o,
                                          bool fast) {
  const int64_t base = (o >> 4) << 4;
  if (fast) {
#pragma unroll
    for (int i = 0; i < NL; ++i) cp_async16(row + 16 * i, llr + base + 16 * i, 16, 0);
  } else {
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      const int64_t a = base + 16 * i;
      const bool ok = (a >= 0) && (a < buf_bytes);
      cp_async16(row + 16 * i, llr + (ok ? a : 0), ok ? 16 : 0, 0);
    }
  }
}

// stage_row split over the T lanes of a window group: lane t copies chunks t, t+T, ...
// (the row is then read by all T lanes: wait for the copies, then __syncwarp)
template <int NL, int T>
__device__ __forceinline__ void stage_row_part(char* row, const int8_t* __restrict__ llr, int64_t buf_bytes,
                                               int64_t o, bool fast, int t) {
  const int64_t base = (o >> 4) << 4;
#pragma unroll
  for (int i0 = 0; i0 < NL; i0 += T) {
    const int i = i0 + t;
    if (i < NL) {
      const int64_t a = base + 16 * i;
      const bool ok = fast || ((a >= 0) && (a < buf_bytes));
      cp_async16(row + 16 * i, llr + (ok ? a : 0), ok ? 16 : 0, 0);
    }
  }
}

// stage_row at byte offset o = o0 + rel (rel 32-bit): the fast path needs no 64-bit
// offset arithmetic beyond one pointer add
template <int NL>
__device__ __forceinline__ void stage_row_rel(char* row, const int8_t* __restrict__ llr, int64_t buf_bytes, int64_t o0,
                                              int rel, bool fast) {
  if (fast) {
    const int8_t* p = reinterpret_cast<const int8_t*>(reinterpret_cast<uintptr_t>(llr + o0 + rel) & ~(uintptr_t)15);
#pragma unroll
    for (int i = 0; i < NL; ++i) cp_async16(row + 16 * i, p + 16 * i, 16, 0);
  } else {
    stage_row<NL>(row, llr, buf_bytes, o0 + rel, false);
  }
}

// NWB words starting at byte `off` (any alignment) of a staged row: NWB+1 aligned 4-byte
// loads and a funnel shift; zero the first zb bytes (stages before the window start)
template <int NWB>
__device__ __forceinline__ void realign_row_at(uint32_t (&out)[NWB], const char* row, int off, int zb) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row + (off & ~3));
  uint32_t v[NWB + 1];
#pragma unroll
  for (int k = 0; k <= NWB; ++k) v[k] = w[k];
  const int r = (off & 3) * 8;
#pragma unroll
  for (int k = 0; k < NWB; ++k) out[k] = __funnelshift_r(v[k], v[k + 1], r);
  if (zb > 0) {
#pragma unroll
    for (int k = 0; k < NWB; ++k) {
      const int lo = zb - 4 * k;
      if (lo >= 4) out[k] = 0u;
      else if (lo > 0) out[k] &= 0xFFFFFFFFu << (8 * lo);
    }
  }
}

// Words [o, o + 4*NWC) of a row staged by stage_row (off = o & 15): NWC+1 aligned
// 4-byte loads and a funnel shift by the byte misalignment; zero the first zb bytes.
template <int NWC>
__device__ __forceinline__ void realign_row(uint32_t (&out)[NWC], const char* row, int off, int zb) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(row + (off & 12));
  uint32_t v[NWC + 1];
#pragma unroll
  for (int k = 0; k <= NWC; ++k) v[k] = w[k];
  const int r = (off & 3) * 8;
#pragma unroll
  for (int k = 0; k < NWC; ++k) out[k] = __funnelshift_r(v[k], v[k + 1], r);
  if (zb > 0) {
#pragma unroll
    for (int k = 0; k < NWC; ++k) {
      const int lo = zb - 4 * k;
      if (lo >= 4) out[k] = 0u;
      else if (lo > 0) out[k] &= 0xFFFFFFFFu << (8 * lo);
    }
  }
}

// LLR byte `byte` of a realigned chunk as (llr << 16), sign-extended.
__device__ __forceinline__ int32_t llr_hi16(uint32_t word, uint32_t sh) {
  // result bytes: [0]=0, [1]=0, [2]=src byte sh, [3]=sign(src byte sh)
  return (int32_t)prmt(word, 0u, ((8u | sh) << 12) | (sh << 8) | 0x44u);
}

// Traceback over the stored BL-stage survivor histories and packed emission of
// the window's emit range [e0, e1) (reference.py:131-144; framing.py:136-137).
// A block's history h holds the decision of block stage p in bit p (newest
// highest); from the state j at the block end:
//   decoded bits of the block = ((h | j << BL) >> (K-1)) & (2^BL - 1)
//   state before the block    = ((j << BL) | h) & (S-1)
// The walk is a state machine so the kernel can interleave one step per
// forward chunk of the next tile (the dependent field loads then hide behind
// ACS work).
template <int K, int BL>
struct Traceback {
  static constexpr uint32_t S = 1u << (K - 1);
  // positions are relative to P0 = floor32(e0), so all bookkeeping is 32-bit
  int64_t wbase;   // absolute word index of relative word 0
  int e0r, e1r;    // relative emit range
  int nr;          // stream end (N) relative, clamped to 2^30
  int top;         // relative word-aligned top of the emitted words
  int gb;          // relative position of block b's first stage
  int hiw;         // next (relative) word to flush; done when < 0
  int lo;          // acc holds decoded bits of relative positions [lo, (hiw+1)*32)
  uint64_t acc;
  uint32_t j;
  int b;           // next block (descending)
  bool active;     // emits output (window exists)
  bool running;    // words left to emit

  __device__ __forceinline__ void start(const Window& g, uint32_t jst, bool act, int nblocks, int64_t N) {
    const int64_t p0 = (g.e0 >> 5) << 5;
    wbase = g.e0 >> 5;
    e0r = (int)(g.e0 - p0);
    e1r = (int)(g.e1 - p0);
    nr = (int)min(N - p0, (int64_t)(1 << 30));
    top = ((e1r + 31) >> 5) << 5;
    hiw = (e1r - 1) >> 5;
    gb = (int)(g.g0 - p0) + BL * (nblocks - 1);
    lo = top;
    acc = 0;
    j = jst;
    b = nblocks - 1;
    active = act;
    running = true;
  }

  __device__ __forceinline__ void flush(const StreamArgs& a) {
    const int wlo = hiw << 5, whi = wlo + 32;
    uint32_t word = (uint32_t)(wlo >= lo ? (acc >> (wlo - lo)) : (acc << (lo - wlo)));
    const int vlo = max(wlo, e0r), vhi = min(whi, e1r);
    const uint32_t mask = (vhi - vlo >= 32) ? 0xFFFFFFFFu : (((1u << (vhi - vlo)) - 1u) << (vlo - wlo));
    word &= mask;
    if (active) {
      const bool owned = (wlo >= e0r) && (min(whi, nr) <= e1r);
      if (owned) a.bits[wbase + hiw] = word;
      else if (word) atomicOr(a.bits + wbase + hiw, word);
    }
    --hiw;
    const int keep = ((hiw + 1) << 5) - lo;
    acc &= (keep >= 64) ? ~0ull : (keep > 0 ? ((1ull << keep) - 1ull) : 0ull);
    running = hiw >= 0;
  }

  // consume block b with history h (0 for blocks that were not stored)
  __device__ __forceinline__ void step(const StreamArgs& a, uint32_t h) {
    uint32_t bits = ((h | (j << BL)) >> (K - 1)) & ((1u << BL) - 1u);
    j = ((j << BL) | h) & (S - 1);
    const int p = gb;
    gb -= BL;
    --b;
    if (p >= top) return;
    const int n_new = lo - p;  // BL, or more/less for the block straddling `top`
    if (n_new < BL) bits &= (1u << n_new) - 1u;
    acc = (acc << n_new) | bits;
    lo = p;
    while (running && (hiw << 5) >= lo) flush(a);
  }

  // blocks below the stored range and words starting before the first chunk
  __device__ __forceinline__ void drain_unstored(const StreamArgs& a) {
    while (running && b >= 0) step(a, 0u);
    while (running) flush(a);
  }
};

// Branch-free traceback step for short history groups (L < K-1 bits per group,
// the 16x2 kernels): each step shifts L decoded bits into a 64-bit register;
// whole words are written by settle(), called once per chunk (<= 43 pending
// bits, so nothing shifts out before it is written).
template <int K, int L>
struct TracebackLite {
  static constexpr uint32_t S = 1u << (K - 1);
  int64_t wbase;   // absolute word index of relative word 0 (P0 = floor32(e0))
  int e0r, e1r, nr;
  int hiw;         // next relative word to write; finished when < 0
  int lo;          // relative position of bit 0 of acc
  uint64_t acc;
  uint32_t j;
  int b;           // next group (descending)
  bool active, running;

  __device__ __forceinline__ void start(const Window& g, uint32_t jst, bool act, int ngroups, int64_t N) {
    const int64_t p0 = (g.e0 >> 5) << 5;
    wbase = g.e0 >> 5;
    e0r = (int)(g.e0 - p0);
    e1r = (int)(g.e1 - p0);
    nr = (int)min(N - p0, (int64_t)(1 << 30));
    hiw = (e1r - 1) >> 5;
    lo = (int)(g.g0 - p0) + L * ngroups;  // window end: nothing accumulated yet
    acc = 0;
    j = jst;
    b = ngroups - 1;
    active = act;
    running = true;
  }
  // consume the history h of group b for the current state j
  __device__ __forceinline__ void step(uint32_t h) {
    const uint32_t bits = (j >> (K - 1 - L)) & ((1u << L) - 1u);  // inputs of the group's stages
    j = ((j << L) | h) & (S - 1);
    acc = (acc << L) | bits;
    lo -= L;
    --b;
  }
  __device__ __forceinline__ void settle(const StreamArgs& a) {
    while (running && (hiw << 5) >= lo) {
      const int wlo = hiw << 5, whi = wlo + 32;
      uint32_t word = (uint32_t)(acc >> (wlo - lo));
      const int vlo = max(wlo, e0r), vhi = min(whi, e1r);
      word &= (vhi - vlo >= 32) ? 0xFFFFFFFFu : (((1u << (vhi - vlo)) - 1u) << (vlo - wlo));
      if (active) {
        if ((wlo >= e0r) && (min(whi, nr) <= e1r)) a.bits[wbase + hiw] = word;
        else if (word) atomicOr(a.bits + wbase + hiw, word);
      }
      --hiw;
      running = hiw >= 0;
    }
  }
  // groups below the stored range (their decisions are never emitted)
  __device__ __forceinline__ void drain_unstored(const StreamArgs& a) {
    while (running && b >= 0) {
      step(0u);
      settle(a);
    }
    if (running) {  // words starting before the window's first group
      while (running) {
        const int wlo = hiw << 5;
        const int sh = lo - wlo;  // > 0: bits below lo are outside the window
        lo = wlo;
        acc = sh < 64 ? acc << sh : 0ull;
        settle(a);
      }
    }
  }
};

// ---------------------------------------------------------------------------
// tcgen05 helpers (tensor-core branch metrics, gen_kernels16.py tc variant).
// Operand tiles are K-major with no swizzle: element (r, k) of an R x 32-byte
// int8 tile at (r/8)*256 + (k/16)*128 + (r%8)*16 + k%16 (8x16-byte core
// matrices; LBO = 128 B between the two K halves, SBO = 256 B between 8-row
// groups).  Checked standalone by tools/tcbm/tc_bm_test.cu.
// ---------------------------------------------------------------------------
namespace tc {
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int kmaj(int r, int k) { return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }
__device__ __forceinline__ uint64_t desc_kmaj(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46);  // version 1 (sm100), SWIZZLE_NONE
}
// kind::i8 instruction descriptor: s32 accumulate, signed int8 A and B, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc) {
  asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
               ::"r"(d_tmem), "l"(da), "l"(db), "r"(idesc), "r"(0));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(phase) : "memory");
  } while (!done);
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void ld4(uint32_t taddr, uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(taddr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// one history group (16 words) of this thread's TMEM lane: columns [taddr, taddr + 16)
__device__ __forceinline__ void st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};"
      ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
template <int COLS>
__device__ __forceinline__ void alloc(uint32_t* dst_smem) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)), "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int COLS>
__device__ __forceinline__ void dealloc(uint32_t taddr) {  // one full warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS));
}
}  // namespace tc

// --- mma.sync register-fragment branch metrics (the 16x2mma form, gen_kernels16.py) ---
namespace mx {
// D = A (16x16 s8, row) . B (16x8 s8, col) + C (s32): a0 rows g, a1 rows g+8 (bytes 4q..4q+3),
// b0 rows 4q..4q+3 of column g, d0/d1 row g cols 2q/2q+1, d2/d3 row g+8 (g = lane/4, q = lane%4)
__device__ __forceinline__ void mma_s8_16816(uint32_t& d0, uint32_t& d1, uint32_t& d2, uint32_t& d3, uint32_t a0,
                                             uint32_t a1, uint32_t b0, uint32_t c) {
  asm("mma.sync.aligned.m16n8k16.row.col.s32.s8.s8.s32 {%0, %1, %2, %3}, {%4, %5}, {%6}, {%7, %7, %7, %7};"
      : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
      : "r"(a0), "r"(a1), "r"(b0), "r"(c));
}
// four 8x8 b16 matrices: lane t holds row t/4, columns 2(t%4), 2(t%4)+1 of matrix i in r_i; lanes
// 8i..8i+7 give the shared addresses of matrix i's rows
__device__ __forceinline__ void stmatrix_x4(uint32_t saddr, uint32_t r0, uint32_t r1, uint32_t r2, uint32_t r3) {
  asm volatile("stmatrix.sync.aligned.m8n8.x4.shared.b16 [%0], {%1, %2, %3, %4};" ::"r"(saddr), "r"(r0), "r"(r1),
               "r"(r2), "r"(r3)
               : "memory");
}
}  // namespace mx

}  // namespace vt
