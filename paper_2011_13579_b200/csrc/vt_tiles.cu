// The paper's tile formulation on real tensor cores: decode_matrix_batch
// (pkg/src/vitertile/matrix.py:277-409, tile.py:61-89) with every 16x16x16 tile op
// D = A x B + C executed as two mma.sync.m16n8k16 (f16 inputs, f32 accumulate).
//
//   A  the tile's +-1 branch-output (BOMAT) blocks (matrix.py:129-265), f16, constant;
//   B  the step's LLRs placed at (b_rows, b_cols) (matrix.py:292-293, 322-323), f16;
//   C  the predecessor path metrics gathered by c_state/c_mask (matrix.py:294, 324);
//   D  candidates: radix-2 rows (i0, i1) per output state, radix-4 four rows, the later
//      candidate winning ties (matrix.py:297-300, 327-333); survivors are the candidate's
//      code (radix-2: 0/1; radix-4: the permuted left local state, perm_tab).
//
// The host packs the reference's tile tables (paper_2011_13579_b200/tiles.py) into
// per-lane fragment tables.  One warp per frame; path metrics and the tile outputs live
// in shared memory.  accumulator="half" reproduces the reference's rounding of every tile
// result to binary16 (tile.py:87-89: f32 accumulate, one rounding): the tensor cores
// accumulate in f32 (exact here: integer LLRs and metrics < 2^24) and the kernel rounds.
// Every warp counts the mma.sync it issues; the counter is the paper's tile-op count.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "../../include/vitertile_b200.h"
#include "vt_internal.h"

namespace {

constexpr int kWarps = 4;  // frames per CTA

struct TileArgs {
  const int8_t* llr;            // (F, N, B) int8
  int64_t F, N;
  int B, S;
  vt_tile_program r2, r4;       // the programs (their tables in device memory; r4 unused for radix 2)
  int radix, half_acc, renormalize;
  uint8_t* surv;                // (F, nsteps, S)
  float* final_lambda;          // (F, S)
  double* offset;               // (F)
  unsigned long long* mma_count;
  int nsteps;
};

__device__ __forceinline__ float round_acc(float v, int half) {
  return half ? __half2float(__float2half_rn(v)) : v;
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1,
                                         const float (&c)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%10, %11, %12, %13};"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(c[0]), "f"(c[1]), "f"(c[2]), "f"(c[3]));
}

__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// one trellis step (1 or 2 stages) of program p for this warp's frame
__device__ void tile_step(const vt_tile_program& p, const float* llr_step, const float* lam, float* lam_new,
                          float* dscr, uint8_t* surv_row, int half, int lane, unsigned long long& mmas) {
  const int g = lane >> 2, q = lane & 3;
  for (int t = 0; t < p.ntiles; ++t) {
    const uint32_t* af = p.a_frag + ((size_t)t * 32 + lane) * 4;
    const uint32_t a[4] = {af[0], af[1], af[2], af[3]};
    const int8_t* bs = p.b_sel + ((size_t)t * 32 + lane) * 8;
    const int16_t* cs = p.c_state + ((size_t)t * 32 + lane) * 8;
    float* d_tile = dscr + t * 256;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      float bv[4], c[4], d[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int s = bs[nb * 4 + i];
        bv[i] = s >= 0 ? llr_step[s] : 0.f;
        const int st = cs[nb * 4 + i];
        c[i] = st >= 0 ? lam[st] : 0.f;
      }
      mma16816(d, a, pack_h2(bv[0], bv[1]), pack_h2(bv[2], bv[3]), c);
      ++mmas;
      const int col = nb * 8 + 2 * q;
      d_tile[g * 16 + col] = round_acc(d[0], half);
      d_tile[g * 16 + col + 1] = round_acc(d[1], half);
      d_tile[(g + 8) * 16 + col] = round_acc(d[2], half);
      d_tile[(g + 8) * 16 + col + 1] = round_acc(d[3], half);
    }
  }
  __syncwarp();
  for (int t = 0; t < p.ntiles; ++t) {
    const float* d_tile = dscr + t * 256;
    for (int o = lane; o < p.nout; o += 32) {
      const size_t oi = (size_t)t * p.nout + o;
      const int st = p.out_state[oi];
      if (st < 0) continue;
      const uint8_t* cand = p.cand + oi * 4;
      float best = d_tile[cand[0]];
      int kb = 0;
      for (int k = 1; k < p.ncand; ++k) {  // the later candidate wins ties (matrix.py:299, 329-330)
        const float v = d_tile[cand[k]];
        if (v >= best) {
          best = v;
          kb = k;
        }
      }
      lam_new[st] = best;
      surv_row[st] = p.code[oi * 4 + kb];
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kWarps * 32) vt_tile_forward(const TileArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t f = (int64_t)blockIdx.x * kWarps + warp;
  const int S = a.S;
  int maxt = a.r2.ntiles;
  if (a.radix == 4 && a.r4.ntiles > maxt) maxt = a.r4.ntiles;
  float* lam0 = smem + (size_t)warp * (2 * S + maxt * 256 + 8);
  float* lam1 = lam0 + S;
  float* dscr = lam1 + S;
  float* llr_s = dscr + maxt * 256;  // the step's (up to 2B <= 8) LLRs
  unsigned long long mmas = 0;
  if (f < a.F) {
    for (int s = lane; s < S; s += 32) lam0[s] = 0.f;
    double off = 0.0;
    const int8_t* fl = a.llr + f * a.N * a.B;
    int64_t t = 0;
    int step = 0;
    __syncwarp();
    while (t < a.N) {
      const bool r4 = a.radix == 4 && t + 1 < a.N;
      const vt_tile_program& p = r4 ? a.r4 : a.r2;
      const int nl = r4 ? 2 * a.B : a.B;
      if (lane < nl) llr_s[lane] = (float)fl[t * a.B + lane];  // LLRs of stages t (and t+1), stage-major
      __syncwarp();
      tile_step(p, llr_s, lam0, lam1, dscr, a.surv + ((size_t)f * a.nsteps + step) * S, a.half_acc, lane, mmas);
      if (a.renormalize) {  // matrix.py:378-382: subtract the per-frame maximum, track it in float64
        float m = -INFINITY;
        for (int s = lane; s < S; s += 32) m = fmaxf(m, lam1[s]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        off += (double)m;
        for (int s = lane; s < S; s += 32) lam1[s] = round_acc(lam1[s] - m, a.half_acc);
        __syncwarp();
      }
      float* tmp = lam0;
      lam0 = lam1;
      lam1 = tmp;
      t += r4 ? 2 : 1;
      ++step;
    }
    for (int s = lane; s < S; s += 32) a.final_lambda[f * S + s] = lam0[s];
    if (lane == 0) a.offset[f] = off;
  }
  if (lane == 0 && mmas) atomicAdd(a.mma_count, mmas);  // (every lane issued the same mma.sync)
}

// matrix._traceback_steps (matrix.py:389-409): from the lowest-index best final state
__global__ void vt_tile_traceback(const uint8_t* surv, const float* final_lambda, const double* offset, int64_t F,
                                  int64_t N, int S, int K, int radix, int nsteps, uint8_t* bits, double* final_metric) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= F) return;
  const float* lam = final_lambda + f * S;
  int j = 0;
  float best = lam[0];
  for (int s = 1; s < S; ++s)
    if (lam[s] > best) {
      best = lam[s];
      j = s;
    }
  final_metric[f] = (double)best + offset[f];  // matrix.py:384
  const int mask2 = (S >> 1) - 1, shift2 = K - 2, mask4 = (1 << (K - 3)) - 1, shift4 = K - 3;
  uint8_t* out = bits + f * N;
  // step k covers stages [t_k, t_k + len): radix-4 steps first, a final radix-2 step when N is odd
  int64_t t_end = N;
  for (int k = nsteps - 1; k >= 0; --k) {
    const bool r4 = radix == 4 && !(k == nsteps - 1 && (N & 1));
    const uint8_t sv = surv[((size_t)f * nsteps + k) * S + j];
    if (!r4) {
      out[t_end - 1] = (uint8_t)(j >> shift2);
      j = 2 * (j & mask2) + sv;
      t_end -= 1;
    } else {
      const int y = j >> shift4;
      out[t_end - 1] = (uint8_t)(y >> 1);
      out[t_end - 2] = (uint8_t)(y & 1);
      j = 4 * (j & mask4) + sv;
      t_end -= 2;
    }
  }
}

}  // namespace

extern "C" {

size_t vt_tile_shared_bytes(int S, int max_tiles) {
  return (size_t)kWarps * (2 * S + max_tiles * 256 + 8) * sizeof(float);
}

int vt_matrix_forward(const vt_code* code, const int8_t* llr, int64_t F, int64_t N, const vt_tile_program* r2,
                      const vt_tile_program* r4, int radix, int half_acc, int renormalize, uint8_t* survivors,
                      float* final_lambda, double* offset, uint8_t* bits, double* final_metric,
                      unsigned long long* mma_count, void* stream) {
  vt_set_error(VT_OK, "");
  if (!code || code->K < 3 || code->K > 9 || code->B < 1 || code->B > 4 || F < 1 || N < 1 || !llr || !r2 ||
      !survivors || !final_lambda || !offset || !bits || !final_metric || !mma_count || (radix != 2 && radix != 4) ||
      (radix == 4 && !r4))
    return vt_set_error(VT_EINVAL, "bad tile-decoder arguments");
  int max_tiles = r2->ntiles;
  if (radix == 4 && r4->ntiles > max_tiles) max_tiles = r4->ntiles;
  if (max_tiles < 1 || max_tiles > 64 || r2->ncand != 2 || (radix == 4 && r4->ncand != 4))
    return vt_set_error(VT_EINVAL, "bad tile program");
  const int S = 1 << (code->K - 1);
  const int nsteps = (int)(radix == 4 ? N / 2 + (N & 1) : N);
  TileArgs a;
  a.llr = llr;
  a.F = F;
  a.N = N;
  a.B = code->B;
  a.S = S;
  a.r2 = *r2;
  a.r4 = radix == 4 ? *r4 : *r2;
  a.radix = radix;
  a.half_acc = half_acc;
  a.renormalize = renormalize;
  a.surv = survivors;
  a.final_lambda = final_lambda;
  a.offset = offset;
  a.mma_count = mma_count;
  a.nsteps = nsteps;
  const size_t smem = vt_tile_shared_bytes(S, max_tiles);
  cudaFuncSetAttribute(vt_tile_forward, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const cudaStream_t s = (cudaStream_t)stream;
  vt_tile_forward<<<(unsigned)((F + kWarps - 1) / kWarps), kWarps * 32, smem, s>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) {
    vt_tile_traceback<<<(unsigned)((F + 127) / 128), 128, 0, s>>>(survivors, final_lambda, offset, F, N, S, code->K,
                                                                    radix, nsteps, bits, final_metric);
    e = cudaGetLastError();
  }
  if (e != cudaSuccess) return vt_set_error(VT_ECUDA, cudaGetErrorString(e));
  return VT_OK;
}

}  // extern "C"
