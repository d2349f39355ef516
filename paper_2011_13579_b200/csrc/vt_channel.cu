// GPU synthetic channel for BER measurement.
//
// Replaces, for BER points, the reference harness's host pipeline
//   channel.generate_bits -> codes.encode_batch -> channel.modulate_awgn
//   (pkg/src/vitertile/channel.py:69-87, codes.py:216-230)
// plus the int8 quantiser the decoder is specified on, fused in one pass, and
// the BER count of channel.compute_ber (channel.py:90-99).
//
// Randomness: counter-based Philox4x32-10 keyed by (seed, point) like the
// reference's Philox streams keyed by (seed, point, purpose) (channel.py:34-35).
// The streams are not numpy's, so GPU BER points agree with the reference in
// distribution (Monte-Carlo confidence intervals), not bit-for-bit; the exact
// path is the host numpy generator + the same GPU decoder.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/vitertile_b200.h"

namespace {

struct Philox {
  __device__ static uint4 round(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
    return make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
  }
  // Philox4x32-10
  __device__ static uint4 gen(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
      c = round(c, k);
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
    return c;
  }
};

__device__ __forceinline__ float u01(uint32_t x) { return ((float)x + 0.5f) * 2.3283064365386963e-10f; }

struct ChannelArgs {
  uint64_t seed;
  uint32_t point;
  int64_t n;          // total stages (frames * frame_len)
  int64_t frame_len;  // encoder restarts from the zero state at every frame start
  int K, B;
  uint32_t gens[VT_MAX_OUTPUTS];
  float sigma, scale;
  int hard;           // 1: hard slicing (llr >= 0 -> +1 else -1), reference.py:202-203
  uint32_t* bits;     // info bits, packed (ceil(n/32) words)
  int8_t* llr;        // (n, B) stage-major
};

// one thread = 32 consecutive stages of the concatenated frame stream
template <int B>
__global__ void __launch_bounds__(256) channel_kernel(const ChannelArgs a) {
  const int64_t word = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p0 = word * 32;
  if (p0 >= a.n) return;
  const uint2 key = make_uint2((uint32_t)a.seed, (uint32_t)(a.seed >> 32) ^ (a.point * 0x9E3779B9u));
  auto info_word = [&](int64_t w) -> uint32_t {
    if (w < 0) return 0u;
    const uint4 r = Philox::gen(make_uint4((uint32_t)w, (uint32_t)(w >> 32), 0u, 0x0B175u), key);
    return r.x;
  };
  uint32_t cur = info_word(word);
  const int64_t valid = min((int64_t)32, a.n - p0);
  if (valid < 32) cur &= (1u << valid) - 1u;
  const uint64_t win = ((uint64_t)cur << 32) | info_word(word - 1);  // bit 32+i = u at stage p0+i
  a.bits[word] = cur;
  const int K = a.K;
  const uint32_t kmask = (1u << K) - 1u;
  uint32_t ow[8 * B];
#pragma unroll
  for (int w = 0; w < 8 * B; ++w) ow[w] = 0u;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < valid) {
      const int64_t p = p0 + i;
      const int64_t hist = p % a.frame_len;  // stages of this frame before p
      uint32_t reg = (uint32_t)(win >> (33 + i - K)) & kmask;  // bit K-1 = u_p, bit 0 = u_{p-K+1}
      if (hist < K - 1) {  // the encoder restarts from the zero state at every frame (codes.py:216-230)
        const int sft = K - 1 - (int)hist;
        reg &= (kmask >> sft) << sft;
      }
      const uint4 r = Philox::gen(make_uint4((uint32_t)p, (uint32_t)(p >> 32), 1u, 0x0A3Cu), key);
      const float rad0 = sqrtf(-2.0f * __logf(u01(r.x))), ang0 = 6.283185307179586f * u01(r.y);
      const float rad1 = sqrtf(-2.0f * __logf(u01(r.z))), ang1 = 6.283185307179586f * u01(r.w);
      float nz[4];
      __sincosf(ang0, &nz[1], &nz[0]);
      __sincosf(ang1, &nz[3], &nz[2]);
      nz[0] *= rad0;
      nz[1] *= rad0;
      nz[2] *= rad1;
      nz[3] *= rad1;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int c = __popc(a.gens[b] & reg) & 1;
        const float y = (1.0f - 2.0f * c) + a.sigma * nz[b];  // BPSK 0 -> +1 (channel.py:83-86)
        int q;
        if (a.hard) q = (y >= 0.0f) ? 1 : -1;
        else q = (int)fminf(fmaxf(rintf(a.scale * y), -127.0f), 127.0f);
        const int idx = i * B + b;
        ow[idx >> 2] |= ((uint32_t)q & 0xFFu) << (8 * (idx & 3));
      }
    }
  }
  uint32_t* dst = reinterpret_cast<uint32_t*>(a.llr + p0 * B);
  const int nw = (int)((valid * B + 3) / 4);
#pragma unroll
  for (int w = 0; w < 8 * B; ++w)
    if (w < nw) dst[w] = ow[w];
}

__global__ void __launch_bounds__(256) count_kernel(const uint32_t* __restrict__ x, const uint32_t* __restrict__ y,
                                                    int64_t nwords, unsigned long long* out) {
  unsigned long long acc = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += (int64_t)gridDim.x * blockDim.x)
    acc += __popc(x[i] ^ y[i]);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
  if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, acc);
}

}  // namespace

extern "C" {

int vt_channel_awgn(const vt_code* code, uint64_t seed, uint32_t point, int64_t frames, int64_t frame_len,
                    float sigma, float llr_scale, int hard, uint32_t* bits, int8_t* llr, void* stream) {
  if (!code || code->K < 2 || code->K > 16 || code->B < 1 || code->B > VT_MAX_OUTPUTS || frames < 1 ||
      frame_len < 1 || !bits || !llr)
    return VT_EINVAL;
  if (code->B < 2 || code->B > 4) return VT_EUNSUPPORTED;
  ChannelArgs a;
  a.seed = seed;
  a.point = point;
  a.n = frames * frame_len;
  a.frame_len = frame_len;
  a.K = code->K;
  a.B = code->B;
  for (int b = 0; b < VT_MAX_OUTPUTS; ++b) a.gens[b] = b < code->B ? code->gens[b] : 0u;
  a.sigma = sigma;
  a.scale = llr_scale;
  a.hard = hard;
  a.bits = bits;
  a.llr = llr;
  const int64_t words = (a.n + 31) / 32;
  const dim3 grid((unsigned)((words + 255) / 256));
  if (a.B == 2) channel_kernel<2><<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  else if (a.B == 3) channel_kernel<3><<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  else channel_kernel<4><<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ECUDA;
}

int vt_count_bit_errors(const uint32_t* a, const uint32_t* b, int64_t nwords, unsigned long long* out,
                        void* stream) {
  if (!a || !b || !out || nwords < 0) return VT_EINVAL;
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), (cudaStream_t)stream);
  if (nwords == 0) return VT_OK;
  int blocks = (int)std::min<int64_t>((nwords + 255) / 256, 148 * 8);
  count_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(a, b, nwords, out);
  return cudaGetLastError() == cudaSuccess ? VT_OK : VT_ECUDA;
}

}  // extern "C"
