// Issue-rate microbenchmark for the integer instructions an ACS (add-compare-select)
// kernel is built from, on sm_100a. Each thread runs NCH independent dependency chains
// so that throughput, not latency, is measured. Reports warp-instructions per cycle
// per SM for each instruction class and for the mixes the decoder uses.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 16
#define ITERS 4096

template <int MODE>
__global__ void __launch_bounds__(256) bench(unsigned* out, unsigned long long* cyc, unsigned seed) {
  unsigned x[NCH];
  unsigned y = seed * 3u + threadIdx.x, z = seed ^ 0x1234567u, m = seed | 1u;
#pragma unroll
  for (int i = 0; i < NCH; ++i) x[i] = seed + i * 77u + threadIdx.x;
  __syncwarp();
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      if (MODE == 0) {  // VIADDMNMX (s32)
        asm volatile("{.reg .s32 t; add.s32 t, %0, %1; max.s32 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(z));
      } else if (MODE == 1) {  // VIADDMNMX.U16x2
        asm volatile("{.reg .b32 t; add.u16x2 t, %0, %1; max.u16x2 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(z));
      } else if (MODE == 2) {  // IMAD 3-register
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(m), "r"(y));
      } else if (MODE == 3) {  // IMAD immediate multiplier
        asm volatile("mad.lo.u32 %0, %0, 3, %1;" : "+r"(x[i]) : "r"(y));
      } else if (MODE == 4) {  // IADD3
        asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(z));
      } else if (MODE == 5) {  // VIADD.16x2
        asm volatile("add.u16x2 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
      } else if (MODE == 6) {  // LOP3
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(y), "r"(z));
      } else if (MODE == 7) {  // PRMT
        asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(x[i]) : "r"(y));
      } else if (MODE == 8) {  // VIMNMX s32
        asm volatile("max.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(y));
      } else if (MODE == 9) {  // radix-2 ACS s32: c1 = x[i^1] + z ; x[i] = max(x[i] + y, c1)
        unsigned c1;
        asm volatile("mad.lo.u32 %0, %1, 1, %2;" : "=r"(c1) : "r"(x[i ^ 1]), "r"(z));
        asm volatile("{.reg .s32 t; add.s32 t, %0, %1; max.s32 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(c1));
      } else if (MODE == 10) {  // radix-2 ACS u16x2: c1 = x[i^1] +16x2 z ; x[i] = max16x2(x[i] + y, c1)
        unsigned c1;
        asm volatile("add.u16x2 %0, %1, %2;" : "=r"(c1) : "r"(x[i ^ 1]), "r"(z));
        asm volatile("{.reg .b32 t; add.u16x2 t, %0, %1; max.u16x2 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(c1));
      } else if (MODE == 11) {  // u16x2 ACS with the carry-free 32-bit add on the FMA pipe
        unsigned c1;
        asm volatile("mad.lo.u32 %0, %1, %3, %2;" : "=r"(c1) : "r"(x[i ^ 1]), "r"(z), "r"(m));
        asm volatile("{.reg .b32 t; add.u16x2 t, %0, %1; max.u16x2 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(c1));
      } else if (MODE == 12) {  // VIMNMX3 s32
        asm volatile("{.reg .s32 t; max.s32 t, %0, %1; max.s32 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(z));
      } else if (MODE == 13) {  // IADD3 + VIADDMNMX (ACS with the add on the ALU pipe)
        unsigned c1;
        asm volatile("{.reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3;}" : "=r"(c1) : "r"(x[i ^ 1]), "r"(z), "r"(m));
        asm volatile("{.reg .s32 t; add.s32 t, %0, %1; max.s32 %0, t, %2;}" : "+r"(x[i]) : "r"(y), "r"(c1));
      }
    }
  }
  unsigned long long t1 = clock64();
  unsigned acc = 0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) acc ^= x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if ((threadIdx.x & 31) == 0) cyc[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = t1 - t0;
}

template <int MODE>
void run(const char* name, int instr_per_chain_iter, int warps_per_sm, int nsm) {
  int threads = 256;
  int blocks_per_sm = warps_per_sm * 32 / threads;
  if (blocks_per_sm < 1) { blocks_per_sm = 1; threads = warps_per_sm * 32; }
  int blocks = nsm * blocks_per_sm;
  int nthreads = blocks * threads, nwarps = nthreads / 32;
  unsigned* out; unsigned long long* cyc;
  cudaMalloc(&out, nthreads * 4); cudaMalloc(&cyc, nwarps * 8);
  bench<MODE><<<blocks, threads>>>(out, cyc, 1);  // warm-up
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<MODE><<<blocks, threads>>>(out, cyc, 7);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long* h = new unsigned long long[nwarps];
  cudaMemcpy(h, cyc, nwarps * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < nwarps; ++i) mx = h[i] > mx ? h[i] : mx;
  double instr_per_warp = (double)ITERS * NCH * instr_per_chain_iter;
  double ipc_sm = instr_per_warp * warps_per_sm / mx;    // warp-instr per cycle per SM
  double mhz = mx / (ms * 1e3);
  printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"warp_instr_per_cycle_per_sm\": %.3f, \"cycles\": %.0f, \"ms\": %.4f, \"implied_mhz\": %.0f}\n",
         name, warps_per_sm, ipc_sm, mx, ms, mhz);
  delete[] h; cudaFree(out); cudaFree(cyc);
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int nsm = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d}\n", p.name, nsm);
  for (int w : {4, 8, 16, 32}) {
    run<0>("VIADDMNMX.s32", 1, w, nsm);
    run<1>("VIADDMNMX.u16x2", 1, w, nsm);
    run<2>("IMAD.3reg", 1, w, nsm);
    run<3>("IMAD.imm", 1, w, nsm);
    run<4>("IADD3", 1, w, nsm);
    run<5>("VIADD.16x2", 1, w, nsm);
    run<6>("LOP3", 1, w, nsm);
    run<7>("PRMT", 1, w, nsm);
    run<8>("VIMNMX.s32", 1, w, nsm);
    run<12>("VIMNMX3.s32", 1, w, nsm);
    run<9>("ACS2_s32(IMAD+VIADDMNMX)", 2, w, nsm);
    run<13>("ACS2_s32(IADD3+VIADDMNMX)", 2, w, nsm);
    run<10>("ACS2_u16x2(VIADD16x2+VIADDMNMX)", 2, w, nsm);
    run<11>("ACS2_u16x2(IMAD+VIADDMNMX)", 2, w, nsm);
  }
  return 0;
}
