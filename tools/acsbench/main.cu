// Host driver for the ACS-rate microbenchmark (tools/acsbench/gen.py).
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#include "acs_bench.cu"

typedef void (*kfn)(const uint32_t*, uint4*, uint32_t*, int);

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  const int nsm = p.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  struct { const char* name; kfn f; int s32; } ks[] = {
    {"v16", acs_v16, 0}, {"v16imad", acs_v16imad, 0}, {"v16g", acs_v16g, 0}, {"v16gi", acs_v16gi, 0}, {"s32", acs_s32, 1}, {"v16gpi", acs_v16gpi, 0}, {"v16gpnci", acs_v16gpnci, 0}};
  const int maxc = 4;
  uint32_t* src; uint4* scratch; uint32_t* out;
  cudaMalloc(&src, (size_t)nsm * maxc * 64 * 128 * 4);
  cudaMemset(src, 0x37, (size_t)nsm * maxc * 64 * 128 * 4);
  cudaMalloc(&scratch, (size_t)nsm * maxc * 128 * 64 * 16);
  cudaMalloc(&out, (size_t)nsm * maxc * 128 * 4);
  const int iters = 2000;
  for (auto& k : ks) {
    cudaFuncSetAttribute((const void*)k.f, cudaFuncAttributeMaxDynamicSharedMemorySize, 0);
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, (const void*)k.f);
    for (int c = 1; c <= 3; ++c) {
      const int grid = nsm * c;
      k.f<<<grid, 128>>>(src, scratch, out, 50);
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k.f<<<grid, 128>>>(src, scratch, out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaError_t err = cudaGetLastError();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      // state updates: 6 stages * 64 states * iters per thread, x2 windows for 16x2
      double su = (double)grid * 128 * iters * 6 * 64 * (k.s32 ? 1 : 2);
      double per_s = su / (ms * 1e-3);
      printf("{\"kernel\": \"%s\", \"ctas_per_sm\": %d, \"regs\": %d, \"ms\": %.3f, \"Gsu_per_s\": %.1f, \"su_per_cycle_per_sm_at_1965\": %.2f, \"err\": \"%s\"}\n",
             k.name, c, fa.numRegs, ms, per_s * 1e-9, per_s / (nsm * 1.965e9), cudaGetErrorString(err));
    }
  }
  return 0;
}
