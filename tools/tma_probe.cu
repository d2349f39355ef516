// Probe: a 3-D TMA tensor map over an int8 LLR stream whose window dimension overlaps
// the line dimension (d0 = 16 bytes, d1 = 16-byte lines, d2 = windows at stride S bytes),
// i.e. the per-window chunk rows of the 16x2 kernels.  Checks that the driver accepts the
// overlapping strides and that one cp.async.bulk.tensor lands box {16, NL, 32} as 32
// consecutive NL*16-byte rows in shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe tools/tma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int NL = 5, ROWS = 32;

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x1, int x2, uint8_t* out) {
  __shared__ alignas(128) uint8_t sm[ROWS * NL * 16];
  __shared__ alignas(8) uint64_t bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(&bar);
  const uint32_t sd = (uint32_t)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(ROWS * NL * 16) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(sd), "l"(&tm), "r"(0), "r"(x1), "r"(x2), "r"(sb) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                 : "=r"(done) : "r"(sb) : "memory");
  for (int i = threadIdx.x; i < ROWS * NL * 16; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int64_t nbytes = 1 << 20, stride = 1024;
  std::vector<uint8_t> h(nbytes);
  for (int64_t i = 0; i < nbytes; ++i) h[i] = (uint8_t)(i * 2654435761u >> 13);
  uint8_t *d, *o;
  cudaMalloc(&d, nbytes);
  cudaMalloc(&o, ROWS * NL * 16);
  cudaMemcpy(d, h.data(), nbytes, cudaMemcpyHostToDevice);
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no entry point\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[3] = {16, (cuuint64_t)(nbytes / 16), (cuuint64_t)((nbytes - 4096) / stride)};
  cuuint64_t strides[2] = {16, (cuuint64_t)stride};
  cuuint32_t box[3] = {16, NL, ROWS}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode overlapping strides: CUresult %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;
  int bad = 0;
  for (int x1 : {0, 3, 7}) {
    for (int x2 : {0, 5}) {
      probe<<<1, 128>>>(tm, x1, x2, o);
      std::vector<uint8_t> got(ROWS * NL * 16);
      cudaError_t e = cudaMemcpy(got.data(), o, got.size(), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
      for (int row = 0; row < ROWS; ++row)
        for (int b = 0; b < NL * 16; ++b) {
          const int64_t src = (int64_t)(x2 + row) * stride + (int64_t)x1 * 16 + b;
          if (got[row * NL * 16 + b] != h[src]) ++bad;
        }
    }
  }
  printf("mismatching bytes: %d\n", bad);
  return bad != 0;
}
