// Standalone check of the tcgen05 int8 MMA plumbing used by the tensor-core
// branch-metric variant: K-major INTERLEAVE (no swizzle) smem descriptors,
// kind::i8 instruction descriptor, TMEM alloc / 32x32b loads, mbarrier commit.
// D[128 x 64] (s32, TMEM) = A[128 x 32] (s8, smem) * B[64 x 32]^T (s8, smem).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, no swizzle: element (r, k) of an R x 32-byte tile at
// (r/8)*256 + (k/16)*128 + (r%8)*16 + (k%16): LBO = 128 B (K halves), SBO = 256 B (8-row groups)
__device__ __forceinline__ int kmaj(int r, int k) { return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address >> 4, bits [0,14)
  d |= (uint64_t)((128 >> 4) & 0x3FFF) << 16;       // leading byte offset (K direction), bits [16,30)
  d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;       // stride byte offset (8-row groups), bits [32,46)
  d |= (uint64_t)1 << 46;                           // version = 1 (sm100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE (bits 61-63)
  return d;
}

__device__ __forceinline__ uint32_t make_idesc_i8(int M, int N) {
  uint32_t d = 0;
  d |= 2u << 4;                 // c_format = S32
  d |= 1u << 7;                 // a_format = signed int8
  d |= 1u << 10;                // b_format = signed int8
  // a_major = b_major = 0 (K-major), no negate
  d |= (uint32_t)(N >> 3) << 17;  // n_dim
  d |= (uint32_t)(M >> 4) << 24;  // m_dim
  return d;
}

__global__ void k(const int8_t* A, const int8_t* B, int* D, int* err) {
  __shared__ __align__(1024) int8_t sA[128 * 32];
  __shared__ __align__(1024) int8_t sB[64 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t mbar;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < 128 * 32; i += 128) sA[kmaj(i / 32, i % 32)] = A[i];
  for (int i = t; i < 64 * 32; i += 128) sB[kmaj(i / 32, i % 32)] = B[i];
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");   // generic smem writes -> async proxy (tensor core)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  if (t == 0) {
    const uint64_t da = make_desc(smem_u32(sA)), db = make_desc(smem_u32(sB));
    const uint32_t id = make_idesc_i8(128, 64);
    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;}"
                 ::"r"(tm), "l"(da), "l"(db), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar)));
  }
  // wait for the MMA (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 64; c0 += 4) {
    uint32_t v0, v1, v2, v3;
    const uint32_t addr = tm + ((uint32_t)(32 * w) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v0), "=r"(v1), "=r"(v2), "=r"(v3) : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    D[t * 64 + c0 + 0] = (int)v0;
    D[t * 64 + c0 + 1] = (int)v1;
    D[t * 64 + c0 + 2] = (int)v2;
    D[t * 64 + c0 + 3] = (int)v3;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(64));
  (void)err;
}

int main() {
  int8_t hA[128 * 32], hB[64 * 32];
  srand(7);
  for (auto& x : hA) x = (int8_t)(rand() % 256 - 128);
  for (auto& x : hB) x = (int8_t)(rand() % 256 - 128);
  int8_t *dA, *dB; int *dD, *derr;
  cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, 128 * 64 * 4); cudaMalloc(&derr, 4);
  cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xFF, 128 * 64 * 4);
  k<<<1, 128>>>(dA, dB, dD, derr);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  static int hD[128 * 64];
  cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      int ref = 0;
      for (int kk = 0; kk < 32; ++kk) ref += (int)hA[m * 32 + kk] * (int)hB[n * 32 + kk];
      if (ref != hD[m * 64 + n]) { if (bad < 5) printf("m=%d n=%d got %d want %d\n", m, n, hD[m * 64 + n], ref); ++bad; }
    }
  printf("mismatches: %d of %d\n", bad, 128 * 64);
  return bad != 0;
}
