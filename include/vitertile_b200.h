/*
 * vitertile_b200 — C ABI of the B200-native framed Viterbi decoder.
 *
 * Drop-in boundary for the reference's decode hot path.  The reference
 * (vitertile 0.1.0, pure Python) has no FFI; its operator boundary is the
 * string dispatch decoder in {"reference","matrix"} plus DecoderConfig
 * (pkg/src/vitertile/framing.py:86-93,111; channel.py:102-110; cli.py:93-97).
 * Every entry point below replaces one reference function on that path:
 *
 *   vt_decode_stream        <- framing.decode_stream / _decode_windows
 *                              (framing.py:86-141) with decoder="reference"
 *                              (reference.decode_batch, reference.py:194-206)
 *   vt_decode_stream_range  <- the same, restricted to windows [w0, w1) of a
 *                              stage sub-range held in device memory (lets the
 *                              host pipeline H2D copies and shard across GPUs)
 *   vt_decode_frames        <- reference.decode_batch (reference.py:194-206):
 *                              F independent frames of N stages, zero initial
 *                              metrics, per-frame final metric
 *   vt_decode_stream_host   <- decode_stream called with HOST buffers (the
 *                              CLI path, cli.py:133-175): H2D, decode, D2H
 *
 * Conventions (all calls):
 *   - Plain pointers and sizes; no allocation inside a call (the caller passes
 *     the workspace sized by vt_workspace_bytes).  Calls are reentrant and
 *     thread-safe; errors are reported per thread.  The only shared state is
 *     append-only: per-(kernel, device) launch facts computed on first use and
 *     the kernels of loaded code modules (vt_load_code_module), both published
 *     with atomics.
 *   - LLRs are int8, stage-major (N, B): element (t, b) at llr[t*B + b], the
 *     layout of the reference CLI's LLR files (cli.py:136-140).  Positive LLR
 *     means the coded bit is more likely 0 (reference.py:28).
 *   - Output bits are packed little-endian: stage t is bit (t & 31) of word
 *     t >> 5 (np.packbits(..., "little"), cli.py:5-6, 170-171).  `bits` must be
 *     zero-initialised by the caller: words shared by two windows are OR-ed.
 *   - Decisions are bit-exact against the reference for integer LLRs: ties
 *     select the second predecessor (reference.py:121), the final state is the
 *     lowest-index argmax (reference.py:138).
 *   - Return 0 on success, a negative VT_E* code on error; vt_last_error()
 *     returns a message for the calling thread.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Kernel form (same bits, different speed): the environment variable
 *     VT_KERNEL_VARIANT = 16x2 | s32 | 16x2tc forces two windows per thread in
 *     packed 16-bit halves (K=8/9: per group of 2/4 lanes), one window per
 *     thread with 32-bit metrics, or 16x2 with tensor-core (tcgen05 kind::i8)
 *     branch metrics (K=7 r1/2); by default 16x2 is used where it exists
 *     (K=7 rate 1/2 and 1/3, K=8, K=9), s32 otherwise (K<=6).
 */
#ifndef VITERTILE_B200_H
#define VITERTILE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VT_MAX_OUTPUTS 8

/* codes.py:51-107 CodeSpec: constraint length K and B generator polynomials
 * (bit K-1 taps the current input bit, bit 0 the oldest register bit). */
typedef struct vt_code {
  int32_t K;
  int32_t B;
  uint32_t gens[VT_MAX_OUTPUTS];
} vt_code;

enum {
  VT_OK = 0,
  VT_EINVAL = -1,      /* bad argument (mirrors the reference's ValueError) */
  VT_EUNSUPPORTED = -2,/* no compiled kernel for this code */
  VT_EWORKSPACE = -3,  /* workspace too small */
  VT_ECUDA = -4        /* CUDA runtime error */
};

/* Library version (major*10000 + minor*100 + patch). */
int vt_version(void);

/* 1 if a compiled sm_100a kernel exists for this code, else 0. */
int vt_code_supported(const vt_code* code);

/* ---- code modules: kernels generated and compiled at run time for codes the
 * library was not built with (the reference decodes any CodeSpec,
 * codes.py:52-107; cli.py:85-90).  paper_2011_13579_b200/jit.py generates the
 * same kernel forms as the build for the new (K, generators), compiles them
 * for sm_100a into a shared library exporting
 *     int vtm_kernels(vt_module_kernel* out, int max);
 * and registers it here.  Module kernels launch through the module (its own
 * CUDA runtime registration); everything else is shared with built-in codes. */
#define VT_MODULE_VERSION 2
typedef int (*vt_module_launch_fn)(const void* stream_args, const void* tensor_map, long long grid,
                                   int no_final_metric, void* stream);
typedef int (*vt_module_prepare_fn)(int* ctas_per_sm);
typedef struct vt_module_kernel {
  int32_t version;                 /* VT_MODULE_VERSION */
  int32_t K, B, T, WPT, SL, CH, BL, SQ, body, rows;
  uint32_t gens[VT_MAX_OUTPUTS];
  int32_t smem, tc, nt, has_nofm;
  vt_module_launch_fn launch;      /* returns a cudaError_t value */
  vt_module_prepare_fn prepare;    /* shared-memory opt-in + occupancy; returns a cudaError_t value */
} vt_module_kernel;

/* Load a code module and register its kernels; returns the number of kernels
 * registered (> 0) or a VT_E* code.  Registered codes stay for the process. */
int vt_load_code_module(const char* path);

/* Message describing the last error on the calling thread ("" if none). */
const char* vt_last_error(void);

/* Workspace (device bytes) needed by vt_decode_stream[_range] / vt_decode_frames
 * for the given geometry on the current device. */
size_t vt_workspace_bytes(const vt_code* code, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1);

/* Decode the whole stream: windows of plan_frames(N, F, V) (framing.py:68-83).
 * llr: device (N, B) int8; bits: device ceil(N/32) uint32 (zeroed);
 * final_metric: optional device int64 per window (max path metric). */
int vt_decode_stream(const vt_code* code, const int8_t* llr, int64_t N, int64_t F, int64_t V, uint32_t* bits,
                     int64_t* final_metric, void* workspace, size_t workspace_bytes, void* stream);

/* Decode windows [w0, w1) of plan_frames(N, F, V).  llr points at stage st0
 * of the stream and holds stages [st0, st1); requires st0 % 16 == 0 (or 0),
 * st0 <= max(0, w0*F - V), st1 >= min(N, min(w1*F, N) + V), llr 16-B aligned.
 * bits is the packed output of the WHOLE stream (word 0 = stages 0..31);
 * final_metric (optional) has w1 - w0 entries. */
int vt_decode_stream_range(const vt_code* code, const int8_t* llr, int64_t st0, int64_t st1, int64_t N, int64_t F,
                           int64_t V, int64_t w0, int64_t w1, uint32_t* bits, int64_t* final_metric,
                           void* workspace, size_t workspace_bytes, void* stream);

/* reference.decode_batch: `frames` independent frames of n stages each,
 * llr device (frames, n, B) int8 (stage-major per frame); bits device packed
 * output of the concatenation (frame f stage t -> bit f*n + t), zeroed;
 * final_metric device int64 per frame (nullable). */
int vt_decode_frames(const vt_code* code, const int8_t* llr, int64_t frames, int64_t n, uint32_t* bits,
                     int64_t* final_metric, void* workspace, size_t workspace_bytes, void* stream);

/* decode_stream with HOST buffers: llr_host (N, B) int8 -> bits_host
 * ceil(N/32) words.  Device staging buffers (llr_dev >= N*B bytes rounded up
 * to 16, bits_dev >= ceil(N/32) words) and the workspace are caller-owned.
 * The copy is pipelined in `nchunks` window ranges on `stream` (synchronous
 * on return).  Pinned host memory gives full PCIe bandwidth. */
int vt_decode_stream_host(const vt_code* code, const int8_t* llr_host, int64_t N, int64_t F, int64_t V,
                          uint32_t* bits_host, int8_t* llr_dev, uint32_t* bits_dev, void* workspace,
                          size_t workspace_bytes, int nchunks, void* stream);

/* Workspace bytes for vt_decode_stream_host over windows [w0, w1) in nchunks
 * pipelined pieces (the maximum over the pieces). */
size_t vt_workspace_bytes_host(const vt_code* code, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1,
                               int nchunks);

/* Shard g of ndev (frames shard with no exchange): out[0..1]
 * = window range [w0, w1), out[2..3] = the stage range [st0, st1) its
 * windows read (V-stage halos; st0 a multiple of 16). */
int vt_shard_range(int64_t N, int64_t F, int64_t V, int ndev, int g, int64_t out[4]);

/* decode_stream with HOST buffers over several devices (framing.decode_stream
 * with workers, framing.py:121-135: the reference fans one stream's windows
 * over threads; here over GPUs).  Shard g (vt_shard_range) runs on
 * devices[g] on its own host thread and stream, pipelined like
 * vt_decode_stream_host: llr_dev[g] holds its stages [st0, st1) (>= (st1 -
 * st0) * B bytes), bits_dev[g] >= ceil(N/32) words, workspace[g] >=
 * vt_workspace_bytes_host(code, N, F, V, w0, w1, nchunks) on that device.
 * Each shard copies the words only it writes straight into bits_host; words
 * two shards share are OR-merged on the host.  A device may appear more than
 * once (separate streams).  Synchronous on return. */
int vt_decode_stream_host_multi(const vt_code* code, const int8_t* llr_host, int64_t N, int64_t F, int64_t V,
                                uint32_t* bits_host, int ndev, const int* devices, int8_t* const* llr_dev,
                                uint32_t* const* bits_dev, void* const* workspace, const size_t* workspace_bytes,
                                int nchunks);

/* ---- the reference's separate forward / traceback stages ----
 * reference.forward_batch (reference.py:95-128): F frames of N stages, llr device
 * (F, N, B) int8; initial_metrics device int64, (S) shared by all frames
 * (init_per_frame = 0), (F, S) per frame (1) or NULL (zeros); renormalize != 0
 * subtracts the per-stage maximum.  Outputs (device): survivors (F, N, S) uint8
 * (1 = the second predecessor won, ties included), final_metrics (F, S) int64,
 * history (F, N, S) int64 per-stage metrics (nullable).  K <= 9. */
int vt_forward_batch(const vt_code* code, const int8_t* llr, int64_t F, int64_t N, const int64_t* initial_metrics,
                     int init_per_frame, int renormalize, uint8_t* survivors, int64_t* final_metrics,
                     int64_t* history, void* stream);

/* reference.traceback_batch (reference.py:131-144): from the lowest-index best
 * final state, bits (F, N) uint8 on the device. */
int vt_traceback_batch(const vt_code* code, const uint8_t* survivors, const int64_t* final_metrics, int64_t F,
                       int64_t N, uint8_t* bits, void* stream);

/* Host helper for reference-style inputs: float64 LLRs (B, N) (row b at
 * llr + b*row_stride) -> int8 stage-major (N, B) in one multithreaded pass
 * (nthreads <= 0: all cores).  VT_EINVAL when a value is not an integer in
 * [-128, 127] (the reference API's float LLRs must be quantised first). */
int vt_pack_llr_f64(const double* llr, int64_t B, int64_t N, int64_t row_stride, int8_t* out, int nthreads);

/* ---- paper-formulation tile decoder with the dragonfly permutation tie order ----
 * matrix.decode_matrix_batch / decode_stream(decoder="matrix") with
 * DecoderConfig(radix=4, optimized=True) (matrix.py:187-265, 306-334, 342-409):
 * two-stage steps whose 4 candidates tie-break by priority prio[f*4 + x]
 * (position of left-local state x of dragonfly f in its group
 * representative's order; higher wins), a final radix-2 step for odd window
 * lengths.  Same stream/window conventions as vt_decode_stream_range; K <= 9. */
size_t vt_workspace_bytes_r4perm(const vt_code* code, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1);
int vt_decode_stream_r4perm(const vt_code* code, const uint8_t* prio, const int8_t* llr, int64_t st0, int64_t st1,
                            int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1, uint32_t* bits,
                            int64_t* final_metric, void* workspace, size_t workspace_bytes, void* stream);

/* ---- the paper's tile formulation on tensor cores ----
 * matrix.decode_matrix_batch (matrix.py:277-409; tile.py:61-89): every tile op
 * D = A x B + C runs as two mma.sync.m16n8k16 (f16 x f16 -> f32).  A program is
 * the reference's pack_radix2 / pack_radix4 tile set (matrix.py:129-265) in
 * per-lane fragment form (built by paper_2011_13579_b200/tiles.py); every
 * table pointer is DEVICE memory, the struct itself is passed by host pointer.
 *   a_frag    [ntiles][32 lanes][4]  A fragment registers (f16x2)
 *   b_sel     [ntiles][32][8]        LLR index of each B fragment element (-1: 0)
 *   c_state   [ntiles][32][8]        path metric of each C fragment element (-1: 0)
 *   cand      [ntiles][nout][4]      candidate D elements (row * 16 + col)
 *   out_state [ntiles][nout]         state each output updates (-1: none)
 *   code      [ntiles][nout][4]      survivor value of each candidate */
typedef struct vt_tile_program {
  int32_t ntiles, nout, ncand, nllr;
  const uint32_t* a_frag;
  const int8_t* b_sel;
  const int16_t* c_state;
  const uint8_t* cand;
  const int16_t* out_state;
  const uint8_t* code;
} vt_tile_program;

/* F frames of N stages, llr device (F, N, B) int8.  radix 2: every step on r2;
 * radix 4: two-stage steps on r4 and a final r2 step for odd N (matrix.py:367-376).
 * half_acc != 0 rounds every tile result to binary16 (accumulator="half");
 * renormalize subtracts each step's maximum (offset, float64, per frame).
 * Device outputs: bits (F, N) uint8 (matrix._traceback_steps), final_metric
 * (F) float64 (max metric + renormalisation offset, matrix.py:384) and
 * *mma_count += the mma.sync instructions issued (2 per 16x16x16 tile op);
 * device scratch: survivors (F, steps, S) uint8, final_lambda (F, S) float32,
 * offset (F) float64 (steps = N for radix 2, ceil(N/2) for radix 4). */
int vt_matrix_forward(const vt_code* code, const int8_t* llr, int64_t F, int64_t N, const vt_tile_program* r2,
                      const vt_tile_program* r4, int radix, int half_acc, int renormalize, uint8_t* survivors,
                      float* final_lambda, double* offset, uint8_t* bits, double* final_metric,
                      unsigned long long* mma_count, void* stream);

/* ---- BER harness (channel.py:69-99 of the reference) ---- */

/* Synthetic AWGN/BPSK frames on the device: `frames` frames of frame_len
 * info bits (Philox4x32-10 keyed by (seed, point)), encoded from the zero
 * state per frame (codes.py:216-230), BPSK 0 -> +1, + sigma * N(0,1)
 * (channel.py:76-87), quantised to int8 LLRs q = clamp(rint(llr_scale * y),
 * -127, 127) (hard != 0: y >= 0 -> +1 else -1, reference.py:202-203).
 * bits: packed info bits (ceil(frames*frame_len/32) words);
 * llr: (frames*frame_len, B) int8, 4-byte aligned.  B must be 2..4. */
int vt_channel_awgn(const vt_code* code, uint64_t seed, uint32_t point, int64_t frames, int64_t frame_len,
                    float sigma, float llr_scale, int hard, uint32_t* bits, int8_t* llr, void* stream);

/* Number of differing bits between two packed device bit vectors
 * (channel.compute_ber, channel.py:90-99); *out is a device counter. */
int vt_count_bit_errors(const uint32_t* a, const uint32_t* b, int64_t nwords, unsigned long long* out,
                        void* stream);

#ifdef __cplusplus
}
#endif

#endif /* VITERTILE_B200_H */
