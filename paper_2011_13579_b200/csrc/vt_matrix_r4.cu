// Radix-4 decode with the dragonfly-group permutation tie order.
//
// Reproduces matrix.decode_matrix_batch(config=DecoderConfig(radix=4, optimized=True))
// (pkg/src/vitertile/matrix.py:187-265 pack_radix4, 306-334 forward_step_radix4,
// 342-386 decode_matrix_batch, 389-409 _traceback_steps) when the group
// optimisation is effective (K=7 171/133): each two-stage step compares the 4
// left states x of a dragonfly in the REPRESENTATIVE's row order, so a tie
// goes to the candidate with the highest position i = perm^-1(x)
// (matrix.py:329-333: "later candidate wins on equality"), not to the highest
// x as in two radix-2 steps.  An odd window length ends with one radix-2 step
// (matrix.py:367-376).
//
// This path is off the headline (the paper-formulation debug decoder), so it
// is a plain thread-per-window kernel: metrics in local memory, branch
// metrics from popc on the fly, 2-bit decisions packed 4 per byte in a global
// scratch slot per thread.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/vitertile_b200.h"

namespace {

struct R4Args {
  const int8_t* llr;
  int64_t st0, st1, N, F, V, w0, w1;
  uint32_t* bits;
  int64_t* final_metric;
  uint8_t* scratch;  // per thread: slot_bytes
  int64_t slot_bytes;
  int K, B;
  uint32_t gens[VT_MAX_OUTPUTS];
  uint8_t prio[64 * 4];  // (S/4) x 4 priority of left-local x in dragonfly f (K <= 9)
};

template <int S>
__global__ void __launch_bounds__(128) r4perm_kernel(const R4Args a) {
  const int K = a.K, B = a.B;
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint8_t* surv = a.scratch + tid * a.slot_bytes;
  int32_t lam[S], nxt[S];
  for (int64_t w = a.w0 + tid; w < a.w1; w += nthreads) {
    const int64_t e0 = w * a.F, e1 = min(e0 + a.F, a.N);
    const int64_t s = max((int64_t)0, e0 - a.V), stop = min(a.N, e1 + a.V);
    const int64_t L = stop - s;
    for (int j = 0; j < S; ++j) lam[j] = 0;
    auto llr = [&](int64_t t, int b) -> int32_t { return (int32_t)a.llr[(s + t - a.st0) * B + b]; };
    auto bm = [&](uint32_t state, uint32_t u, int64_t t) -> int32_t {  // reference.py:79-82 branch metric
      const uint32_t reg = (u << (K - 1)) | state;
      int32_t d = 0;
      for (int b = 0; b < B; ++b) d += (__popc(a.gens[b] & reg) & 1) ? -llr(t, b) : llr(t, b);
      return d;
    };
    const int64_t nsteps4 = L / 2;
    const bool odd = (L & 1) != 0;
    const uint32_t fmask = (uint32_t)(S / 4 - 1);
    for (int64_t st = 0; st < nsteps4; ++st) {
      const int64_t t = 2 * st;
      uint8_t* sv = surv + st * (S / 4);
      for (int J = 0; J < S; J += 4) {
        uint32_t packed = 0;
        for (int jj = 0; jj < 4; ++jj) {
          const uint32_t j = (uint32_t)(J + jj);
          const uint32_t f = j & fmask, u2 = j >> (K - 2), u1 = (j >> (K - 3)) & 1u;
          int32_t best = 0;
          int bprio = -1, bx = 0;
          for (int x = 0; x < 4; ++x) {
            const uint32_t i = 4 * f + (uint32_t)x;
            const uint32_t mid = (u1 << (K - 2)) | (i >> 1);
            const int32_t m = lam[i] + bm(i, u1, t) + bm(mid, u2, t + 1);
            const int pr = a.prio[f * 4 + x];
            if (bprio < 0 || m > best || (m == best && pr > bprio)) {
              best = m;
              bprio = pr;
              bx = x;
            }
          }
          nxt[j] = best;
          packed |= (uint32_t)bx << (2 * jj);
        }
        sv[J / 4] = (uint8_t)packed;
      }
      for (int j = 0; j < S; ++j) lam[j] = nxt[j];
    }
    if (odd) {  // final radix-2 step, natural tie rule (take1 = cand1 >= cand0)
      const int64_t t = L - 1;
      uint8_t* sv = surv + nsteps4 * (S / 4);
      for (int J = 0; J < S; J += 4) {
        uint32_t packed = 0;
        for (int jj = 0; jj < 4; ++jj) {
          const uint32_t j = (uint32_t)(J + jj), u = j >> (K - 2), i0 = 2 * (j & (S / 2 - 1));
          const int32_t c0 = lam[i0] + bm(i0, u, t), c1 = lam[i0 + 1] + bm(i0 + 1, u, t);
          nxt[j] = c1 >= c0 ? c1 : c0;
          packed |= (uint32_t)(c1 >= c0) << (2 * jj);
        }
        sv[J / 4] = (uint8_t)packed;
      }
      for (int j = 0; j < S; ++j) lam[j] = nxt[j];
    }
    uint32_t js = 0;
    for (int j = 1; j < S; ++j)
      if (lam[j] > lam[js]) js = (uint32_t)j;
    if (a.final_metric) a.final_metric[w - a.w0] = lam[js];
    // traceback (matrix.py:389-409), emitting [e0, e1)
    uint32_t word = 0;
    int64_t cur_w = -1;
    auto put = [&](int64_t pos, uint32_t bit) {
      if (pos < e0 || pos >= e1) return;
      const int64_t wi = pos >> 5;
      if (wi != cur_w) {
        if (cur_w >= 0 && word) atomicOr(a.bits + cur_w, word);
        cur_w = wi;
        word = 0;
      }
      word |= bit << (pos & 31);
    };
    int64_t t = L;
    if (odd) {
      t = L - 1;
      const uint32_t d = (surv[nsteps4 * (S / 4) + js / 4] >> (2 * (js & 3))) & 1u;
      put(s + t, js >> (K - 2));
      js = 2 * (js & (S / 2 - 1)) + d;
    }
    for (int64_t st = nsteps4 - 1; st >= 0; --st) {
      t = 2 * st;
      const uint32_t x = (surv[st * (S / 4) + js / 4] >> (2 * (js & 3))) & 3u;
      const uint32_t y = js >> (K - 3);
      put(s + t + 1, y >> 1);
      put(s + t, y & 1u);
      js = 4 * (js & (uint32_t)(S / 4 - 1)) + x;
      if (s + t <= e0) break;
    }
    if (cur_w >= 0 && word) atomicOr(a.bits + cur_w, word);
  }
}

constexpr int kThreads = 128;

int64_t grid_for(int64_t nwin) {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return std::max<int64_t>(1, std::min<int64_t>((nwin + kThreads - 1) / kThreads, (int64_t)sms * 4));
}

int64_t slot_bytes(int K, int64_t N, int64_t F, int64_t V) {
  const int64_t L = std::min<int64_t>(N, F + 2 * V);
  return ((L / 2 + 1) * ((1 << (K - 1)) / 4) + 15) / 16 * 16;
}

}  // namespace

extern "C" {

size_t vt_workspace_bytes_r4perm(const vt_code* code, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1) {
  if (!code || code->K < 3 || code->K > 9 || N < 1 || F < 1 || V < 0 || w1 <= w0) return 0;
  return (size_t)(grid_for(w1 - w0) * kThreads * slot_bytes(code->K, N, F, V));
}

int vt_decode_stream_r4perm(const vt_code* code, const uint8_t* prio, const int8_t* llr, int64_t st0, int64_t st1,
                            int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1, uint32_t* bits,
                            int64_t* final_metric, void* workspace, size_t workspace_bytes, void* stream) {
  if (!code || !prio || !llr || !bits || code->K < 3 || code->K > 9 || code->B < 1 || code->B > VT_MAX_OUTPUTS)
    return VT_EINVAL;
  if (N < 1 || F < 1 || V < 0 || w0 < 0 || w1 <= w0 || w1 > (N + F - 1) / F) return VT_EINVAL;
  if (st0 > std::max<int64_t>(0, w0 * F - V) || st1 < std::min<int64_t>(N, std::min<int64_t>(w1 * F, N) + V))
    return VT_EINVAL;
  if (workspace_bytes < vt_workspace_bytes_r4perm(code, N, F, V, w0, w1) || !workspace) return VT_EWORKSPACE;
  R4Args a;
  a.llr = llr;
  a.st0 = st0;
  a.st1 = st1;
  a.N = N;
  a.F = F;
  a.V = V;
  a.w0 = w0;
  a.w1 = w1;
  a.bits = bits;
  a.final_metric = final_metric;
  a.scratch = (uint8_t*)workspace;
  a.slot_bytes = slot_bytes(code->K, N, F, V);
  a.K = code->K;
  a.B = code->B;
  for (int b = 0; b < VT_MAX_OUTPUTS; ++b) a.gens[b] = b < code->B ? code->gens[b] : 0u;
  const int S = 1 << (code->K - 1);
  for (int i = 0; i < 64 * 4; ++i) a.prio[i] = i < S ? prio[i] : 0;
  const dim3 grid((unsigned)grid_for(w1 - w0));
  cudaStream_t s = (cudaStream_t)stream;
  switch (code->K) {
    case 3: r4perm_kernel<4><<<grid, kThreads, 0, s>>>(a); break;
    case 4: r4perm_kernel<8><<<grid, kThreads, 0, s>>>(a); break;
    case 5: r4perm_kernel<16><<<grid, kThreads, 0, s>>>(a); break;
    case 6: r4perm_kernel<32><<<grid, kThreads, 0, s>>>(a); break;
    case 7: r4perm_kernel<64><<<grid, kThreads, 0, s>>>(a); break;
    case 8: r4perm_kernel<128><<<grid, kThreads, 0, s>>>(a); break;
    default: r4perm_kernel<256><<<grid, kThreads, 0, s>>>(a); break;
  }
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ECUDA;
}

}  // extern "C"
