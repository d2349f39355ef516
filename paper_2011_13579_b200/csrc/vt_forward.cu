// reference.forward_batch / traceback_batch (pkg/src/vitertile/reference.py:95-144) on the GPU.
//
// The decode path fuses the ACS recursion and the traceback (vt_capi.cu); these two
// entry points expose the separate stages of the reference API, with their full
// outputs: per-stage survivor decisions (F, N, S) uint8, final metrics (F, S) and,
// optionally, the per-stage metric history (F, N, S).  Exact in int64 for integer
// LLRs (reference.py:111-128: cand0/cand1 from pred0/pred1 + llr . sgn, take1 =
// cand1 >= cand0, optional renormalisation by the per-stage maximum).
//
// forward: one CTA per frame, one thread per state, metrics double-buffered in
// shared memory (survivor and history writes are coalesced over the states).
// traceback: one thread per frame.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/vitertile_b200.h"

namespace {

struct FwdArgs {
  const int8_t* llr;  // (F, N, B)
  int64_t F, N;
  const int64_t* init;  // (S) or (F, S) or null
  int init_per_frame;
  int renormalize;
  uint8_t* surv;      // (F, N, S)
  int64_t* lam_out;   // (F, S)
  int64_t* hist;      // (F, N, S) or null
  int K, B;
  uint32_t gens[VT_MAX_OUTPUTS];
};

__global__ void forward_kernel(const FwdArgs a) {
  extern __shared__ int64_t sm[];
  const int S = blockDim.x;
  const int j = threadIdx.x;
  const int64_t f = blockIdx.x;
  int64_t* lam = sm;          // [2][S]
  int64_t* red = sm + 2 * S;  // [S / 32] warp maxima
  lam[j] = a.init ? a.init[(a.init_per_frame ? f * S : 0) + j] : 0;
  const uint32_t half = (uint32_t)S / 2;
  const uint32_t i0 = 2u * ((uint32_t)j & (half - 1u)), i1 = i0 + 1u;
  const uint32_t u = (uint32_t)j >> (a.K - 2);
  const uint32_t reg0 = (u << (a.K - 1)) | i0, reg1 = (u << (a.K - 1)) | i1;
  // branch-output signs of the two candidates (reference.py:79-82): +l for output 0, -l for 1
  uint32_t neg0 = 0, neg1 = 0;
  for (int b = 0; b < a.B; ++b) {
    neg0 |= (uint32_t)(__popc(a.gens[b] & reg0) & 1) << b;
    neg1 |= (uint32_t)(__popc(a.gens[b] & reg1) & 1) << b;
  }
  __syncthreads();
  const int8_t* llr = a.llr + f * a.N * a.B;
  int cur = 0;
  for (int64_t t = 0; t < a.N; ++t) {
    int64_t d0 = 0, d1 = 0;
    for (int b = 0; b < a.B; ++b) {
      const int64_t l = llr[t * a.B + b];
      d0 += ((neg0 >> b) & 1u) ? -l : l;
      d1 += ((neg1 >> b) & 1u) ? -l : l;
    }
    const int64_t c0 = lam[cur * S + i0] + d0, c1 = lam[cur * S + i1] + d1;
    const bool take1 = c1 >= c0;
    int64_t v = take1 ? c1 : c0;
    a.surv[(f * a.N + t) * S + j] = take1 ? 1 : 0;
    if (a.renormalize) {  // lam -= max over states (reference.py:124-125)
      int64_t m = v;
      for (int o = 16; o > 0; o >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xFFFFFFFFu, m, o));
      if (S > 32) {
        if ((j & 31) == 0) red[j >> 5] = m;
        __syncthreads();
        m = red[0];
        for (int w = 1; w < S / 32; ++w) m = max(m, red[w]);
      }
      v -= m;
    }
    lam[(cur ^ 1) * S + j] = v;
    if (a.hist) a.hist[(f * a.N + t) * S + j] = v;
    cur ^= 1;
    __syncthreads();
  }
  a.lam_out[f * S + j] = lam[cur * S + j];
}

// S < 32: shuffles over a partial warp need the active-lane mask; run those codes with
// one full warp where lanes >= S idle (they compute but never write)
__global__ void forward_kernel_small(const FwdArgs a, int S) {
  __shared__ int64_t lam[2][32];
  const int j = threadIdx.x;
  const bool live = j < S;
  const int64_t f = blockIdx.x;
  const int js = live ? j : 0;
  lam[0][j] = live ? (a.init ? a.init[(a.init_per_frame ? f * S : 0) + j] : 0) : 0;
  const uint32_t half = (uint32_t)S / 2;
  const uint32_t i0 = 2u * ((uint32_t)js & (half - 1u)), i1 = i0 + 1u;
  const uint32_t u = (uint32_t)js >> (a.K - 2);
  const uint32_t reg0 = (u << (a.K - 1)) | i0, reg1 = (u << (a.K - 1)) | i1;
  uint32_t neg0 = 0, neg1 = 0;
  for (int b = 0; b < a.B; ++b) {
    neg0 |= (uint32_t)(__popc(a.gens[b] & reg0) & 1) << b;
    neg1 |= (uint32_t)(__popc(a.gens[b] & reg1) & 1) << b;
  }
  __syncwarp();
  const int8_t* llr = a.llr + f * a.N * a.B;
  int cur = 0;
  for (int64_t t = 0; t < a.N; ++t) {
    int64_t d0 = 0, d1 = 0;
    for (int b = 0; b < a.B; ++b) {
      const int64_t l = llr[t * a.B + b];
      d0 += ((neg0 >> b) & 1u) ? -l : l;
      d1 += ((neg1 >> b) & 1u) ? -l : l;
    }
    const int64_t c0 = lam[cur][i0] + d0, c1 = lam[cur][i1] + d1;
    const bool take1 = c1 >= c0;
    int64_t v = take1 ? c1 : c0;
    if (live) a.surv[(f * a.N + t) * S + j] = take1 ? 1 : 0;
    if (a.renormalize) {
      int64_t m = live ? v : INT64_MIN;
      for (int o = 16; o > 0; o >>= 1) m = max(m, (int64_t)__shfl_xor_sync(0xFFFFFFFFu, m, o));
      v -= m;
    }
    lam[cur ^ 1][j] = v;
    if (live && a.hist) a.hist[(f * a.N + t) * S + j] = v;
    cur ^= 1;
    __syncwarp();
  }
  if (live) a.lam_out[f * S + j] = lam[cur][j];
}

// traceback_batch (reference.py:131-144): j = argmax (lowest index on ties), then
// out[t] = j >> (K-2); j = 2 (j & mask) + surv[t][j]
__global__ void traceback_kernel(const uint8_t* __restrict__ surv, const int64_t* __restrict__ lam, int64_t F,
                                 int64_t N, int K, uint8_t* __restrict__ bits) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const int S = 1 << (K - 1);
  uint32_t j = 0;
  int64_t best = lam[f * S];
  for (int s = 1; s < S; ++s)
    if (lam[f * S + s] > best) {
      best = lam[f * S + s];
      j = (uint32_t)s;
    }
  const uint32_t mask = (uint32_t)S / 2 - 1u;
  for (int64_t t = N - 1; t >= 0; --t) {
    bits[f * N + t] = (uint8_t)(j >> (K - 2));
    j = 2u * (j & mask) + surv[(f * N + t) * S + j];
  }
}

}  // namespace

extern "C" {

int vt_forward_batch(const vt_code* code, const int8_t* llr, int64_t F, int64_t N, const int64_t* initial_metrics,
                     int init_per_frame, int renormalize, uint8_t* survivors, int64_t* final_metrics,
                     int64_t* history, void* stream) {
  if (!code || !llr || !survivors || !final_metrics || code->K < 3 || code->K > 9 || code->B < 1 ||
      code->B > VT_MAX_OUTPUTS || F < 0 || N < 0)
    return VT_EINVAL;
  if (F == 0) return VT_OK;
  FwdArgs a;
  a.llr = llr;
  a.F = F;
  a.N = N;
  a.init = initial_metrics;
  a.init_per_frame = init_per_frame;
  a.renormalize = renormalize;
  a.surv = survivors;
  a.lam_out = final_metrics;
  a.hist = history;
  a.K = code->K;
  a.B = code->B;
  for (int b = 0; b < VT_MAX_OUTPUTS; ++b) a.gens[b] = b < code->B ? code->gens[b] : 0u;
  const int S = 1 << (code->K - 1);
  cudaStream_t s = (cudaStream_t)stream;
  if (S >= 32) {
    forward_kernel<<<(unsigned)F, S, (size_t)(2 * S + S / 32) * sizeof(int64_t), s>>>(a);
  } else {
    forward_kernel_small<<<(unsigned)F, 32, 0, s>>>(a, S);
  }
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ECUDA;
}

int vt_traceback_batch(const vt_code* code, const uint8_t* survivors, const int64_t* final_metrics, int64_t F,
                       int64_t N, uint8_t* bits, void* stream) {
  if (!code || !survivors || !final_metrics || !bits || code->K < 3 || code->K > 9 || F < 0 || N < 0)
    return VT_EINVAL;
  if (F == 0 || N == 0) return VT_OK;
  traceback_kernel<<<(unsigned)((F + 127) / 128), 128, 0, (cudaStream_t)stream>>>(survivors, final_metrics, F, N,
                                                                                   code->K, bits);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ECUDA;
}

}  // extern "C"
