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
  int nc;                 // 16-stage chunks per window (uniform for the launch)
  int b_lo;               // first chunk whose histories are stored
  int nbs;                // stored chunks per window (nc - b_lo)
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

// max(a + b, c): ptxas fuses add.s32 + max.s32 into one DPX VIADDMNMX (ALU pipe)
__device__ __forceinline__ int32_t addmax(int32_t a, int32_t b, int32_t c) {
  int32_t d;
  asm("{.reg .s32 t; add.s32 t, %1, %2; max.s32 %0, t, %3;}" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

// Window geometry of window w (framing.py:78-82) in the end-aligned chunk frame.
struct Window {
  int64_t e0, e1;   // emit range
  int64_t s, stop;  // window range
  int64_t g0;       // stream stage of chunk 0 (= stop - 16*nc; may be < s: zero padding)
};

__device__ __forceinline__ Window window_geometry(const StreamArgs& a, int64_t w) {
  Window g;
  g.e0 = w * a.F;
  g.e1 = min(g.e0 + a.F, a.N);
  g.s = max((int64_t)0, g.e0 - a.V);
  g.stop = min(a.N, g.e1 + a.V);
  g.g0 = g.stop - 16 * (int64_t)a.nc;
  return g;
}

// Load the 16-byte words covering LLR bytes [o, o + 16B) of the buffer (o may
// be negative or run past the end: those words read as zero).
template <int B>
__device__ __forceinline__ void load_raw(uint4 (&raw)[B + 1], const int8_t* __restrict__ llr, int64_t buf_bytes,
                                         int64_t o) {
  const int64_t base = (o >> 4) << 4;  // floor to 16 (arithmetic shift)
#pragma unroll
  for (int i = 0; i <= B; ++i) {
    const int64_t a = base + 16 * i;
    if (a >= 0 && a < buf_bytes)
      raw[i] = __ldg(reinterpret_cast<const uint4*>(llr + a));
    else
      raw[i] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// Realign raw words by the byte misalignment (0..15) into 4B words holding
// bytes [o, o + 16B); zero the first `zb` bytes (stages before the window).
template <int B>
__device__ __forceinline__ void realign(uint32_t (&out)[4 * B], const uint4 (&raw)[B + 1], int shift, int zb) {
  constexpr int NW = 4 * (B + 1);
  uint32_t w[NW];
#pragma unroll
  for (int i = 0; i <= B; ++i) {
    w[4 * i + 0] = raw[i].x;
    w[4 * i + 1] = raw[i].y;
    w[4 * i + 2] = raw[i].z;
    w[4 * i + 3] = raw[i].w;
  }
  const int q = shift >> 2, r = (shift & 3) * 8;
#pragma unroll
  for (int i = 0; i + 1 < NW; ++i) w[i] = (q & 1) ? w[i + 1] : w[i];
#pragma unroll
  for (int i = 0; i + 2 < NW; ++i) w[i] = (q & 2) ? w[i + 2] : w[i];
#pragma unroll
  for (int k = 0; k < 4 * B; ++k) out[k] = __funnelshift_r(w[k], w[k + 1], r);
  if (zb > 0) {
#pragma unroll
    for (int k = 0; k < 4 * B; ++k) {
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

// Traceback over the stored 16-stage survivor histories and packed emission of
// the window's emit range [e0, e1) (reference.py:131-144; framing.py:136-137).
//   jst: final state (lowest-index argmax);  field(b, j) returns the 16-bit
//   history of state j at the end of chunk b (decision of stage p in bit p).
// Per chunk: bits = ((h | j << 16) >> (K-1)) & 0xFFFF, j = h & (S-1).
template <int K, class FieldFn>
__device__ __forceinline__ void traceback_emit(const StreamArgs& a, const Window& g, uint32_t jst, bool active,
                                               FieldFn field) {
  constexpr uint32_t S = 1u << (K - 1);
  const int64_t top = ((g.e1 + 31) >> 5) << 5;
  int64_t hiw = (g.e1 - 1) >> 5;
  const int64_t loww = g.e0 >> 5;
  int64_t lo = top;  // acc holds the decoded bits of stream positions [lo, (hiw + 1) * 32)
  uint64_t acc = 0;
  auto flush = [&]() {
    const int64_t wlo = hiw << 5, whi = wlo + 32;
    uint32_t word = (uint32_t)(wlo >= lo ? (acc >> (wlo - lo)) : (acc << (lo - wlo)));
    const int64_t vlo = max(wlo, g.e0), vhi = min(whi, g.e1);
    const uint32_t mask = (vhi - vlo >= 32) ? 0xFFFFFFFFu : (((1u << (vhi - vlo)) - 1u) << (vlo - wlo));
    word &= mask;
    if (active) {
      const bool owned = (wlo >= g.e0) && (min(whi, a.N) <= g.e1);
      if (owned) a.bits[hiw] = word;
      else if (word) atomicOr(a.bits + hiw, word);
    }
    --hiw;
    const int64_t keep = ((hiw + 1) << 5) - lo;
    acc &= (keep >= 64) ? ~0ull : (keep > 0 ? ((1ull << keep) - 1ull) : 0ull);
  };
  for (int b = a.nc - 1; b >= 0 && hiw >= loww; --b) {
    const int64_t gb = g.g0 + 16 * (int64_t)b;
    const uint32_t h = (b >= a.b_lo) ? field(b - a.b_lo, jst) : 0u;
    uint32_t bits16 = ((h | (jst << 16)) >> (K - 1)) & 0xFFFFu;
    jst = h & (S - 1);
    if (gb >= top) continue;
    const int n_new = (int)(lo - gb);  // 16, or less for the block straddling `top`
    if (n_new < 16) bits16 &= (1u << n_new) - 1u;
    acc = (acc << n_new) | bits16;
    lo = gb;
    while (hiw >= loww && (hiw << 5) >= lo) flush();
  }
  // words that start before the window's first chunk (only their in-window bits are kept)
  while (hiw >= loww) flush();
}

}  // namespace vt
