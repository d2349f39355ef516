// C ABI of the B200 framed Viterbi decoder (see include/vitertile_b200.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <dlfcn.h>
#include <mutex>
#include <string>
#include <cmath>
#include <thread>
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/vitertile_b200.h"
#include "vt_common.cuh"
#include "vt_internal.h"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

}  // namespace

int vt_set_error(int code, const char* msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  return fail(VT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

// (threads per CTA: KernelEntry::nt)

struct Geometry {
  int64_t nwin;
  int nc, b_lo, nbs;
};

Geometry geometry(int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1, int CH, int BL) {
  // windows are cut into CH-stage chunks aligned to the window end; survivor
  // histories are stored per BL-stage group (BL divides CH)
  Geometry g;
  g.nwin = w1 - w0;
  const int64_t lmax = std::min<int64_t>(N, F + 2 * V);
  g.nc = (int)((lmax + CH - 1) / CH);
  const int64_t ng = (int64_t)g.nc * (CH / BL);
  const int64_t head = std::min<int64_t>(N, F + V);  // max (stop - emit_start) over windows
  int64_t blo = ((int64_t)CH * g.nc - head) / BL;     // first group any window needs for its emit range
  if (blo < 0) blo = 0;
  g.b_lo = (int)blo;
  g.nbs = (int)(ng - blo);
  return g;
}

// ---------------------------------------------------------------------------
// kernel registry: one generated kernel per supported code (gen/registry.inc)
// ---------------------------------------------------------------------------
struct KernelEntry {
  int K, B, T, WPT, SL, CH, BL, SQ;
  int body;  // stages per loop body of the 16x2 forms (the unit of the leading-padding skip); 0 for s32
  int rows;  // > 0: the kernel takes a TMA tensor map of its LLR chunk rows (16-byte lines per row)
  uint32_t gens[VT_MAX_OUTPUTS];
  const void* fn;
  const void* fn_nofm;  // variant without final-metric bookkeeping (nullptr: use fn)
  int smem;             // dynamic shared memory bytes per CTA
  int tc;               // 1: tcgen05 / 2: mma.sync branch-metric variant (opt-in); 3: TMEM history window
  int nt;               // threads per CTA
  // kernels of a runtime-loaded code module (vt_load_code_module) launch through the module,
  // which carries its own CUDA runtime registration of them
  vt_module_launch_fn launch;
  vt_module_prepare_fn prepare;
};

#define VT_KERNEL(fn_, fnnf_, smem_, tc_, nt_, K_, B_, T_, WPT_, SL_, CH_, BL_, SQ_, BODY_, ROWS_, ...) \
  {K_, B_, T_, WPT_, SL_, CH_, BL_, SQ_, BODY_, ROWS_, __VA_ARGS__, (const void*)&fn_, (const void*)(fnnf_), smem_, tc_, nt_, \
   nullptr, nullptr},
}  // namespace
#include "gen/registry_decl.inc"
namespace {

const KernelEntry* registry(int* n) {
  static const KernelEntry table[] = {
#include "gen/registry.inc"
  };
  *n = (int)(sizeof(table) / sizeof(table[0]));
  return table;
}

// Kernels of runtime-loaded code modules (vt_load_code_module): appended under a lock,
// published by the release store of g_ndyn, never removed (entries stay valid).  1024 entries:
// ~400 distinct run-time codes per process (64 ran out after ~25 codes in tools/stress_codes.py).
constexpr int kMaxDyn = 1024;
KernelEntry g_dyn[kMaxDyn];
std::atomic<int> g_ndyn{0};
std::mutex g_dyn_mu;

// Kernel variant: "16x2" (two windows per thread -- per group of 2/4 lanes for K=8/9 --
// in packed 16-bit halves), "s32" (one window per thread, 32-bit metrics) or "16x2tc"
// (16x2 with the branch metrics of each 12-stage chunk computed on the tensor cores:
// tcgen05 kind::i8, the paper's LLR x codeword-matrix contraction) or "16x2mma" (the same
// contraction per body with mma.sync.m16n8k16 s8 register fragments; tc = 2).  Default: 16x2
// where it exists with 3-bit history groups (measured fastest for every such code);
// s32 otherwise.  VT_KERNEL_VARIANT forces one.
int variant_rank(const KernelEntry* e, const char* env) {
  // lower is better; entries of the requested variant win, then the default order
  const bool is16 = e->WPT > 1, istc = e->tc == 1 || e->tc == 2;  // (tc 3: TMEM history window, a default form)
  if (env && strcmp(env, "16x2tc") == 0) return e->tc == 1 ? 0 : (is16 && !istc ? 1 : 2);
  if (env && strcmp(env, "16x2mma") == 0) return e->tc == 2 ? 0 : (is16 && !istc ? 1 : 2);
  if (env && strcmp(env, "16x2") == 0) return (is16 && !istc) ? 0 : (istc ? 2 : 1);
  if (env && strcmp(env, "s32") == 0) return is16 ? 2 : 0;
  if (istc) return 3;                       // opt-in only
  // 16x2 preferred wherever 3-bit history groups fit (K=7 r1/2: 163 vs 118 Gbps; K=7 r1/3
  // with exact-minimum renormalisation: 127.5 vs 113 -- 143.4 with the subset minimum; K=9 over
  // 4 lanes: 32.3 vs 25.1 -- 36.8 with the subset minimum)
  if (is16) return e->BL >= 3 ? 0 : 2;
  return 1;
}

const KernelEntry* find(const vt_code* c) {
  if (!c) return nullptr;
  const char* env = getenv("VT_KERNEL_VARIANT");
  int n;
  const KernelEntry* t = registry(&n);
  const int nd = g_ndyn.load(std::memory_order_acquire);
  const KernelEntry* best = nullptr;
  for (int i = 0; i < n + nd; ++i) {
    const KernelEntry* e = i < n ? &t[i] : &g_dyn[i - n];
    if (e->K != c->K || e->B != c->B) continue;
    bool same = true;
    for (int b = 0; b < c->B; ++b) same = same && e->gens[b] == c->gens[b];
    if (!same) continue;
    if (!best || variant_rank(e, env) < variant_rank(best, env)) best = e;
  }
  return best;
}

// index of an entry in [static table, dynamic table] (per-entry launch caches)
int entry_index(const KernelEntry* k) {
  int n = 0;
  const KernelEntry* t = registry(&n);
  if (k >= t && k < t + n) return (int)(k - t);
  if (k >= g_dyn && k < g_dyn + kMaxDyn) return n + (int)(k - g_dyn);
  return -1;
}

int validate(const vt_code* c) {
  if (!c) return fail(VT_EINVAL, "code is NULL");
  if (c->K < 3 || c->K > 16) return fail(VT_EINVAL, "constraint length %d out of range", c->K);
  if (c->B < 2 || c->B > VT_MAX_OUTPUTS) return fail(VT_EINVAL, "need 2..%d generators, got %d", VT_MAX_OUTPUTS, c->B);
  for (int b = 0; b < c->B; ++b)
    if (c->gens[b] >= (1u << c->K)) return fail(VT_EINVAL, "generator %o does not fit in %d bits", c->gens[b], c->K);
  return VT_OK;
}

// Per (kernel entry, device) launch facts, computed once: the dynamic shared memory
// opt-in (cudaFuncSetAttribute) and the CTA capacity sms * occupancy.  Small calls
// (one frame) are host-bound, so these stay off the per-call path.
constexpr int kMaxEntries = 64 + kMaxDyn, kMaxDevices = 64;
std::atomic<int> g_cap[kMaxEntries][kMaxDevices];  // 0: not yet computed

int current_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
  return dev;
}

// opt the kernels into their dynamic shared memory (above the 48 KB default); idempotent.
// Returns the CTAs per SM the kernel can hold.
int prepare(const KernelEntry* k) {
  int occ = 1;
  if (k->prepare) {
    if (k->prepare(&occ) != 0 || occ < 1) occ = 1;
    return occ;
  }
  if (k->smem > 0) {
    cudaFuncSetAttribute(k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem);
    if (k->fn_nofm) cudaFuncSetAttribute(k->fn_nofm, cudaFuncAttributeMaxDynamicSharedMemorySize, k->smem);
  }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k->fn, k->nt, k->smem);
  if (getenv("VT_DEBUG_OCC")) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k->fn);
    fprintf(stderr, "[vt] occupancy K=%d tc=%d: %d CTAs/SM (err %d, regs %d, static smem %zu, dyn %d, max dyn %d)\n", k->K,
            k->tc, occ, (int)e, fa.numRegs, fa.sharedSizeBytes, k->smem, fa.maxDynamicSharedSizeBytes);
  }
  if (e != cudaSuccess || occ < 1) occ = 1;
  if ((k->tc == 1 || k->tc == 3) && e == cudaSuccess) {
    // The occupancy query answers 1 for the tcgen05 kernels although two CTAs fit (256 TMEM
    // columns each, 2 x ~77 KB shared memory, <= 240 registers): size by those limits.
    cudaFuncAttributes fa;
    if (cudaFuncGetAttributes(&fa, k->fn) == cudaSuccess && fa.numRegs > 0) {
      const int by_regs = 65536 / (((fa.numRegs + 7) / 8) * 8 * k->nt);
      const int by_smem = (228 * 1024) / (k->smem + (int)fa.sharedSizeBytes + 1024);
      occ = std::max(occ, std::min({by_regs, by_smem, 2}));
    }
  }
  return occ;
}

// CTAs that run concurrently on the device (prepares the kernel on first use per device)
int64_t cta_capacity(const KernelEntry* k) {
  const char* env = getenv("VT_CTAS_PER_SM");
  const int idx = entry_index(k);
  const int dev = current_device();
  const bool cacheable = !(env && atoi(env) > 0) && idx >= 0 && idx < kMaxEntries && dev < kMaxDevices;
  if (cacheable) {
    const int c = g_cap[idx][dev].load(std::memory_order_acquire);
    if (c > 0) return c;
  }
  int occ = prepare(k);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (env && atoi(env) > 0) occ = atoi(env);
  const int cap = sms * std::min(occ, 4);
  if (cacheable) g_cap[idx][dev].store(cap, std::memory_order_release);
  return cap;
}

int64_t grid_for(const KernelEntry* k, int64_t nwin) {
  const int64_t wpc = (int64_t)k->nt * k->WPT / k->T;  // windows per CTA
  const int64_t tiles = (nwin + wpc - 1) / wpc;
  const int64_t cap = cta_capacity(k);
  return std::max<int64_t>(1, std::min(tiles, cap));
}

int64_t window_len(int64_t N, int64_t F, int64_t V, int64_t w) {
  const int64_t e0 = w * F, e1 = std::min(e0 + F, N);
  return std::min(N, e1 + V) - std::max<int64_t>(0, e0 - V);
}

// Leading-padding hazard.  The 16x2 kernels trace tile i back while they run tile i+1
// forward and skip up to CH/body bodies of leading zero padding per window; a skip of more
// than b_lo history groups would let tile i+1's history stores overtake tile i's traceback
// fetches (gen_kernels16.py).  Windows at least min(N, F + V) long never need such a skip
// (b_lo is sized by that length), so only a suffix of short tail windows can (the window
// length is non-increasing over the stream tail: a short last window, V = 0).
bool skip_hazard(const KernelEntry* k, const Geometry& g, int64_t N, int64_t F, int64_t V, int64_t w) {
  if (k->WPT <= 1 || k->body <= 0) return false;
  const int chb = k->CH / k->body, gpb = k->body / k->BL;
  const int64_t skip = std::min<int64_t>(chb, std::max<int64_t>(0, (int64_t)k->CH * g.nc - window_len(N, F, V, w)) /
                                                  k->body);
  return skip * gpb > g.b_lo;
}

// First window of the hazardous suffix of [w0, w1) (w1 when there is none).
int64_t hazard_start(const KernelEntry* k, const Geometry& g, int64_t N, int64_t F, int64_t V, int64_t w0,
                     int64_t w1) {
  int64_t wh = w1;
  while (wh > w0 && skip_hazard(k, g, N, F, V, wh - 1)) --wh;
  return wh;
}

// One launch = the persistent grid over [w0, wh) and, when the range ends in hazardous short
// windows, a second launch over [wh, w1) with one tile per CTA (no CTA decodes a tile after
// another there).  The kernels stay unchanged (a runtime cap on the skip measured 2.6% slower
// on the headline).  Scratch is reused by the second launch (stream order).
struct LaunchPlan {
  int64_t wh;          // split point
  int64_t grid_main;   // CTAs of [w0, wh) (0: empty)
  int64_t grid_tail;   // CTAs of [wh, w1) (0: empty)
};

LaunchPlan plan_launch(const KernelEntry* k, const Geometry& g, int64_t N, int64_t F, int64_t V, int64_t w0,
                       int64_t w1) {
  LaunchPlan p;
  p.wh = hazard_start(k, g, N, F, V, w0, w1);
  const int64_t wpc = (int64_t)k->nt * k->WPT / k->T;  // windows per CTA tile
  p.grid_main = p.wh > w0 ? grid_for(k, p.wh - w0) : 0;
  p.grid_tail = w1 > p.wh ? (w1 - p.wh + wpc - 1) / wpc : 0;
  return p;
}

size_t scratch_bytes(const KernelEntry* k, const Geometry& g, int64_t grid) {
  return (size_t)grid * g.nbs * k->SQ * k->nt * sizeof(uint4);
}

size_t plan_scratch(const KernelEntry* k, const Geometry& g, const LaunchPlan& p) {
  return scratch_bytes(k, g, std::max(p.grid_main, p.grid_tail));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda
// dependency: the library also loads on machines without a driver, e.g. to size workspaces)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// The 16x2 kernels' TMA view of the launch's LLR buffer: lines of 16 bytes, and rows (a warp's
// same-parity windows) 2*F*B bytes apart; box = one chunk row of `rows` lines for 32 windows.
// Returns false (the kernels then stage per thread) when the geometry does not allow it.
bool encode_rows_map(const KernelEntry* k, const vt::StreamArgs& a, CUtensorMap* map) {
  if (k->rows <= 0 || getenv("VT_NO_TMA")) return false;
  const int64_t stride = 2 * a.F * k->B, buf_bytes = (a.st1 - a.st0) * k->B;
  if (stride % 16 != 0 || stride >= ((int64_t)1 << 40) || buf_bytes < 16) return false;
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t dims[3] = {16, (cuuint64_t)(buf_bytes / 16), 32};
  const cuuint64_t strides[2] = {16, (cuuint64_t)stride};
  const cuuint32_t box[3] = {16, (cuuint32_t)k->rows, 32}, es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(a.llr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch(const KernelEntry* k, vt::StreamArgs a, int64_t w0, int64_t w1, int64_t grid, void* stream) {
  if (w1 <= w0 || grid <= 0) return VT_OK;
  if (a.final_metric) a.final_metric += (w0 - a.w0);
  a.w0 = w0;
  a.w1 = w1;
  alignas(64) CUtensorMap map;
  memset(&map, 0, sizeof(map));
  a.tma = encode_rows_map(k, a, &map) ? 1 : 0;
  const bool nofm = a.final_metric == nullptr && k->fn_nofm;
  if (k->launch) {
    const int e = k->launch(&a, &map, (long long)grid, nofm ? 1 : 0, stream);
    if (e != 0) return cuda_fail((cudaError_t)e, "kernel launch (code module)");
    return VT_OK;
  }
  void* args[] = {&a, &map};
  const void* fn = nofm ? k->fn_nofm : k->fn;
  cudaError_t e = cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(k->nt), args, (size_t)k->smem, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return VT_OK;
}

}  // namespace

extern "C" {

int vt_version(void) { return 100; }

const char* vt_last_error(void) { return g_err; }

int vt_code_supported(const vt_code* code) { return find(code) != nullptr ? 1 : 0; }

int vt_load_code_module(const char* path) {
  g_err[0] = 0;
  if (!path) return fail(VT_EINVAL, "module path is NULL");
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) return fail(VT_EINVAL, "cannot load code module %s: %s", path, dlerror());
  auto entries = reinterpret_cast<int (*)(vt_module_kernel*, int)>(dlsym(h, "vtm_kernels"));
  if (!entries) return fail(VT_EINVAL, "%s does not export vtm_kernels", path);
  vt_module_kernel mk[16];
  const int n = entries(mk, 16);
  if (n < 1 || n > 16) return fail(VT_EINVAL, "%s: bad kernel count %d", path, n);
  std::lock_guard<std::mutex> lock(g_dyn_mu);
  int nd = g_ndyn.load(std::memory_order_relaxed);
  if (nd + n > kMaxDyn) return fail(VT_EINVAL, "too many code modules loaded");
  for (int i = 0; i < n; ++i) {
    const vt_module_kernel& m = mk[i];
    if (m.version != VT_MODULE_VERSION || !m.launch || !m.prepare)
      return fail(VT_EINVAL, "%s: kernel %d has an incompatible descriptor", path, i);
    KernelEntry& e = g_dyn[nd + i];
    e.K = m.K; e.B = m.B; e.T = m.T; e.WPT = m.WPT; e.SL = m.SL; e.CH = m.CH; e.BL = m.BL; e.SQ = m.SQ;
    e.body = m.body;
    e.rows = m.rows;
    for (int b = 0; b < VT_MAX_OUTPUTS; ++b) e.gens[b] = m.gens[b];
    e.fn = nullptr;
    e.fn_nofm = m.has_nofm ? reinterpret_cast<const void*>(1) : nullptr;  // (a flag: the module picks the function)
    e.smem = m.smem; e.tc = m.tc; e.nt = m.nt;
    e.launch = m.launch;
    e.prepare = m.prepare;
  }
  g_ndyn.store(nd + n, std::memory_order_release);
  return n;
}

size_t vt_workspace_bytes(const vt_code* code, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1) {
  const KernelEntry* k = find(code);
  if (!k || N < 1 || F < 1 || V < 0 || w1 <= w0) return 0;
  const Geometry g = geometry(N, F, V, w0, w1, k->CH, k->BL);
  cta_capacity(k);
  return plan_scratch(k, g, plan_launch(k, g, N, F, V, w0, w1));
}

int vt_decode_stream_range(const vt_code* code, const int8_t* llr, int64_t st0, int64_t st1, int64_t N, int64_t F,
                           int64_t V, int64_t w0, int64_t w1, uint32_t* bits, int64_t* final_metric,
                           void* workspace, size_t workspace_bytes, void* stream) {
  g_err[0] = 0;
  int rc = validate(code);
  if (rc) return rc;
  const KernelEntry* k = find(code);
  if (!k)
    return fail(VT_EUNSUPPORTED, "no sm_100a kernel compiled for K=%d B=%d generators (%o, %o, ...)", code->K,
                code->B, code->gens[0], code->gens[1]);
  if (N < 1) return fail(VT_EINVAL, "stream must have at least one stage");
  if (F < 1) return fail(VT_EINVAL, "frame length must be >= 1");
  if (V < 0) return fail(VT_EINVAL, "overlap must be >= 0");
  const int64_t nw_total = (N + F - 1) / F;
  if (w0 < 0 || w1 > nw_total || w0 >= w1) return fail(VT_EINVAL, "window range [%lld, %lld) outside [0, %lld)",
                                                      (long long)w0, (long long)w1, (long long)nw_total);
  if (!llr || !bits) return fail(VT_EINVAL, "llr and bits must be device pointers");
  if (((uintptr_t)llr & 15) != 0) return fail(VT_EINVAL, "llr must be 16-byte aligned");
  if (st0 != 0 && (st0 % 16) != 0) return fail(VT_EINVAL, "st0 must be a multiple of 16");
  const int64_t need_lo = std::max<int64_t>(0, w0 * F - V);
  const int64_t need_hi = std::min<int64_t>(N, std::min<int64_t>(w1 * F, N) + V);
  if (st0 > need_lo || st1 < need_hi || st1 > N)
    return fail(VT_EINVAL, "llr stage range [%lld, %lld) does not cover [%lld, %lld)", (long long)st0,
                (long long)st1, (long long)need_lo, (long long)need_hi);

  const Geometry g = geometry(N, F, V, w0, w1, k->CH, k->BL);
  cta_capacity(k);  // (prepared once per device)
  const LaunchPlan p = plan_launch(k, g, N, F, V, w0, w1);
  const size_t need = plan_scratch(k, g, p);
  if (!workspace || workspace_bytes < need)
    return fail(VT_EWORKSPACE, "workspace %zu bytes < required %zu", workspace_bytes, need);

  vt::StreamArgs a;
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
  a.scratch = reinterpret_cast<uint4*>(workspace);
  a.nc = g.nc;
  a.b_lo = g.b_lo;
  a.nbs = g.nbs;
  a.tma = 0;
  rc = launch(k, a, w0, p.wh, p.grid_main, stream);
  if (rc) return rc;
  return launch(k, a, p.wh, w1, p.grid_tail, stream);
}

int vt_decode_stream(const vt_code* code, const int8_t* llr, int64_t N, int64_t F, int64_t V, uint32_t* bits,
                     int64_t* final_metric, void* workspace, size_t workspace_bytes, void* stream) {
  if (F < 1) return fail(VT_EINVAL, "frame length must be >= 1");
  if (N < 1) return fail(VT_EINVAL, "stream must have at least one stage");
  return vt_decode_stream_range(code, llr, 0, N, N, F, V, 0, (N + F - 1) / F, bits, final_metric, workspace,
                                workspace_bytes, stream);
}

int vt_decode_frames(const vt_code* code, const int8_t* llr, int64_t frames, int64_t n, uint32_t* bits,
                     int64_t* final_metric, void* workspace, size_t workspace_bytes, void* stream) {
  if (frames < 1 || n < 1) return fail(VT_EINVAL, "need frames >= 1 and n >= 1");
  // F independent frames == a stream of frames*n stages cut with F=n, V=0
  return vt_decode_stream(code, llr, frames * n, n, 0, bits, final_metric, workspace, workspace_bytes, stream);
}

int vt_pack_llr_f64(const double* llr, int64_t B, int64_t N, int64_t row_stride, int8_t* out, int nthreads) {
  if (!llr || !out || B < 1 || N < 0 || row_stride < N) return fail(VT_EINVAL, "bad LLR buffer geometry");
  if (nthreads < 1) nthreads = (int)std::min<unsigned>(32u, std::max(1u, std::thread::hardware_concurrency()));
  const int64_t per = std::max<int64_t>(1 << 16, (N + nthreads - 1) / nthreads);
  std::atomic<int64_t> bad{-1};  // lowest offending stage seen (any), -1 if none
  // Branch-free, vectorisable block pass (one contiguous row at a time, 4K-stage blocks so
  // the interleaved int8 block stays cached across the B rows); a block that holds an
  // offending value is rescanned for its first one.  (Was a per-element std::rint call:
  // 1.4 GB/s per thread.)
  auto first_bad = [&](int64_t t0, int64_t t1) -> int64_t {
    for (int64_t t = t0; t < t1; ++t)
      for (int64_t b = 0; b < B; ++b) {
        const double v = llr[b * row_stride + t];
        if (!(v >= -128.0 && v <= 127.0) || (double)(int)v != v) return t;
      }
    return -1;
  };
  auto work = [&](int64_t t0, int64_t t1) {
    constexpr int64_t BLK = 4096;
    for (int64_t c0 = t0; c0 < t1; c0 += BLK) {
      const int64_t c1 = std::min(t1, c0 + BLK);
      int okall = 1;
      for (int64_t b = 0; b < B; ++b) {
        const double* __restrict__ src = llr + b * row_stride;
        int8_t* __restrict__ dst = out + b;
        int ok = 1;
        for (int64_t t = c0; t < c1; ++t) {
          const double v = src[t];
          const bool in = (v >= -128.0) & (v <= 127.0);  // false for NaN
          const double c = in ? v : 0.0;
          const int iv = (int)c;
          ok &= (int)(in & ((double)iv == c));
          dst[t * B] = (int8_t)iv;
        }
        okall &= ok;
      }
      if (!okall) {
        const int64_t e0 = first_bad(c0, c1);
        int64_t e = bad.load();
        while ((e < 0 || e0 < e) && !bad.compare_exchange_weak(e, e0)) {}
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int64_t t0 = per; t0 < N; t0 += per) pool.emplace_back(work, t0, std::min(N, t0 + per));
  work(0, std::min(N, per));
  for (auto& th : pool) th.join();
  if (bad.load() >= 0)
    return fail(VT_EINVAL, "LLR at stage %lld is not an integer in [-128, 127] (int8-quantised LLRs; use "
                "quantize_llr)", (long long)bad.load());
  return VT_OK;
}

}  // extern "C"

namespace {

// Shard g of G: contiguous balanced window range and the stage range (V-stage halos,
// st0 floored to 16) its windows read (sharding.shard_windows mirrors this).
void shard_range(int64_t N, int64_t F, int64_t V, int64_t G, int64_t g, int64_t* w0, int64_t* w1, int64_t* st0,
                 int64_t* st1) {
  const int64_t nw = (N + F - 1) / F;
  *w0 = nw * g / G;
  *w1 = nw * (g + 1) / G;
  *st0 = (std::max<int64_t>(0, *w0 * F - V) / 16) * 16;
  *st1 = *w1 > *w0 ? std::min<int64_t>(N, std::min<int64_t>(*w1 * F, N) + V) : *st0;
}

// Output words of window range [w0, w1): [own_lo, own_hi) hold only its bits; edge[0] /
// edge[1] (index or -1) are the words it shares with the previous / next range.
struct WordRange {
  int64_t own_lo, own_hi, edge[2];
};

WordRange word_range(int64_t N, int64_t F, int64_t w0, int64_t w1) {
  WordRange r;
  const int64_t e0 = w0 * F, e1 = std::min(w1 * F, N), nwords = (N + 31) / 32;
  r.own_lo = (e0 + 31) / 32;
  r.own_hi = e1 == N ? nwords : e1 / 32;
  r.edge[0] = (e0 % 32) ? e0 / 32 : -1;
  r.edge[1] = (e1 < N && (e1 % 32)) ? e1 / 32 : -1;
  if (r.edge[0] >= 0 && r.edge[0] == r.edge[1]) r.edge[1] = -1;  // one word shared with both neighbours
  if (r.own_hi < r.own_lo) r.own_hi = r.own_lo;
  return r;
}

// Windows [w0, w1) from host LLRs, pipelined in nchunks window ranges: H2D on one copy
// stream, the decode on `s`, D2H of the words only this range writes into bits_host on a
// second copy stream; the shared edge words go to edge_out (merged by the caller).
// llr_dev holds stages from dst0 (multiple of 16); bits_dev is indexed by stream word.
int host_range(const vt_code* code, const int8_t* llr_host, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1,
               uint32_t* bits_host, int8_t* llr_dev, int64_t dst0, uint32_t* bits_dev, void* workspace,
               size_t workspace_bytes, int nchunks, cudaStream_t s, uint32_t edge_out[2]) {
  const int B = code->B;
  const int64_t nw = w1 - w0;
  if (nchunks < 1) nchunks = 1;
  if (nchunks > nw) nchunks = (int)nw;
  const WordRange wr = word_range(N, F, w0, w1);
  // copy and compute run on separate streams so chunk i+1's H2D overlaps chunk i's decode
  // (created per call on the current device: the call is a whole-range decode, and
  // nothing outlives it)
  cudaStream_t cs_in = nullptr, cs_out = nullptr;
  if (cudaStreamCreateWithFlags(&cs_in, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&cs_out, cudaStreamNonBlocking) != cudaSuccess) {
    if (cs_in) cudaStreamDestroy(cs_in);
    return fail(VT_ECUDA, "cannot create copy streams");
  }
  const int64_t mlo = (w0 * F) / 32, mhi = (std::min(w1 * F, N) + 31) / 32;
  int rc = 0;
  cudaError_t e = cudaMemsetAsync(bits_dev + mlo, 0, (size_t)(mhi - mlo) * 4, s);
  if (e != cudaSuccess) rc = cuda_fail(e, "memset");
  cudaEvent_t ev_start;
  cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
  cudaEventRecord(ev_start, s);
  cudaStreamWaitEvent(cs_in, ev_start, 0);
  cudaStreamWaitEvent(cs_out, ev_start, 0);

  int64_t copied_hi = 0, words_done = wr.own_lo;
  for (int i = 0; i < nchunks && rc == 0; ++i) {
    const int64_t c0w = w0 + nw * i / nchunks, c1w = w0 + nw * (i + 1) / nchunks;
    const int64_t st0 = (std::max<int64_t>(0, c0w * F - V) / 16) * 16;
    const int64_t st1 = std::min<int64_t>(N, std::min<int64_t>(c1w * F, N) + V);
    const int64_t c0 = std::max(st0, copied_hi);
    if (st1 > c0) {
      e = cudaMemcpyAsync(llr_dev + (c0 - dst0) * B, llr_host + c0 * B, (size_t)(st1 - c0) * B, cudaMemcpyHostToDevice,
                          cs_in);
      if (e != cudaSuccess) { rc = cuda_fail(e, "H2D"); break; }
      copied_hi = st1;
    }
    cudaEvent_t ev_in, ev_k;
    cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_k, cudaEventDisableTiming);
    cudaEventRecord(ev_in, cs_in);
    cudaStreamWaitEvent(s, ev_in, 0);
    rc = vt_decode_stream_range(code, llr_dev + (st0 - dst0) * B, st0, st1, N, F, V, c0w, c1w, bits_dev, nullptr,
                                workspace, workspace_bytes, s);
    cudaEventRecord(ev_k, s);
    cudaStreamWaitEvent(cs_out, ev_k, 0);
    // words complete after this chunk: all below the next chunk's first emit word
    const int64_t wend = (i + 1 == nchunks) ? wr.own_hi : std::min<int64_t>(wr.own_hi, std::min(N, c1w * F) / 32);
    if (rc == 0 && wend > words_done) {
      e = cudaMemcpyAsync(bits_host + words_done, bits_dev + words_done, (size_t)(wend - words_done) * 4,
                          cudaMemcpyDeviceToHost, cs_out);
      if (e != cudaSuccess) rc = cuda_fail(e, "D2H");
      words_done = wend;
    }
    cudaEventDestroy(ev_in);
    cudaEventDestroy(ev_k);
  }
  cudaEvent_t ev_done;
  cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
  cudaEventRecord(ev_done, cs_out);
  cudaStreamWaitEvent(s, ev_done, 0);
  e = cudaStreamSynchronize(s);
  cudaEventDestroy(ev_done);
  cudaEventDestroy(ev_start);
  cudaStreamDestroy(cs_in);
  cudaStreamDestroy(cs_out);
  if (rc == 0 && e != cudaSuccess) rc = cuda_fail(e, "decode_stream_host");
  for (int k = 0; k < 2 && rc == 0; ++k) {
    edge_out[k] = 0;
    if (wr.edge[k] >= 0) {
      e = cudaMemcpy(&edge_out[k], bits_dev + wr.edge[k], 4, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) rc = cuda_fail(e, "edge word");
    }
  }
  return rc;
}

int check_host_args(const vt_code* code, int64_t N, int64_t F, int64_t V, const void* llr_host, const void* bits_host) {
  int rc = validate(code);
  if (rc) return rc;
  if (!find(code)) return fail(VT_EUNSUPPORTED, "no sm_100a kernel compiled for this code");
  if (N < 1 || F < 1 || V < 0) return fail(VT_EINVAL, "bad geometry");
  if (!llr_host || !bits_host) return fail(VT_EINVAL, "NULL buffer");
  return VT_OK;
}

}  // namespace

extern "C" {

int vt_decode_stream_host(const vt_code* code, const int8_t* llr_host, int64_t N, int64_t F, int64_t V,
                          uint32_t* bits_host, int8_t* llr_dev, uint32_t* bits_dev, void* workspace,
                          size_t workspace_bytes, int nchunks, void* stream) {
  g_err[0] = 0;
  int rc = check_host_args(code, N, F, V, llr_host, bits_host);
  if (rc) return rc;
  if (!llr_dev || !bits_dev) return fail(VT_EINVAL, "NULL buffer");
  uint32_t edge[2];
  return host_range(code, llr_host, N, F, V, 0, (N + F - 1) / F, bits_host, llr_dev, 0, bits_dev, workspace,
                    workspace_bytes, nchunks, (cudaStream_t)stream, edge);
}

int vt_shard_range(int64_t N, int64_t F, int64_t V, int ndev, int g, int64_t out[4]) {
  g_err[0] = 0;
  if (N < 1 || F < 1 || V < 0 || ndev < 1 || g < 0 || g >= ndev || !out) return fail(VT_EINVAL, "bad shard request");
  shard_range(N, F, V, ndev, g, &out[0], &out[1], &out[2], &out[3]);
  return VT_OK;
}

size_t vt_workspace_bytes_host(const vt_code* code, int64_t N, int64_t F, int64_t V, int64_t w0, int64_t w1,
                               int nchunks) {
  const int64_t nw = w1 - w0;
  if (nw <= 0) return 0;
  if (nchunks < 1) nchunks = 1;
  if (nchunks > nw) nchunks = (int)nw;
  size_t need = 0;
  for (int i = 0; i < nchunks; ++i) {
    const int64_t c0 = w0 + nw * i / nchunks, c1 = w0 + nw * (i + 1) / nchunks;
    if (c1 > c0) need = std::max(need, vt_workspace_bytes(code, N, F, V, c0, c1));
  }
  return need;
}

int vt_decode_stream_host_multi(const vt_code* code, const int8_t* llr_host, int64_t N, int64_t F, int64_t V,
                                uint32_t* bits_host, int ndev, const int* devices, int8_t* const* llr_dev,
                                uint32_t* const* bits_dev, void* const* workspace, const size_t* workspace_bytes,
                                int nchunks) {
  g_err[0] = 0;
  int rc = check_host_args(code, N, F, V, llr_host, bits_host);
  if (rc) return rc;
  if (ndev < 1 || ndev > 64 || !devices || !llr_dev || !bits_dev || !workspace || !workspace_bytes)
    return fail(VT_EINVAL, "bad device list");
  for (int g = 0; g < ndev; ++g)
    if (!llr_dev[g] || !bits_dev[g]) return fail(VT_EINVAL, "NULL device buffer for shard %d", g);
  std::vector<int> rcs(ndev, 0);
  std::vector<std::string> msgs(ndev);
  std::vector<uint32_t> edges(2 * ndev, 0);
  std::vector<int64_t> edge_idx(2 * ndev, -1);
  auto work = [&](int g) {
    int64_t w0, w1, st0, st1;
    shard_range(N, F, V, ndev, g, &w0, &w1, &st0, &st1);
    if (w1 <= w0) return;
    const WordRange wr = word_range(N, F, w0, w1);
    edge_idx[2 * g] = wr.edge[0];
    edge_idx[2 * g + 1] = wr.edge[1];
    cudaError_t e = cudaSetDevice(devices[g]);
    if (e != cudaSuccess) { rcs[g] = cuda_fail(e, "cudaSetDevice"); msgs[g] = g_err; return; }
    cudaStream_t s = nullptr;
    e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) { rcs[g] = cuda_fail(e, "stream"); msgs[g] = g_err; return; }
    rcs[g] = host_range(code, llr_host, N, F, V, w0, w1, bits_host, llr_dev[g], st0, bits_dev[g], workspace[g],
                        workspace_bytes[g], nchunks, s, &edges[2 * g]);
    if (rcs[g]) msgs[g] = g_err;
    cudaStreamDestroy(s);
  };
  std::vector<std::thread> pool;
  for (int g = 1; g < ndev; ++g) pool.emplace_back(work, g);
  {
    int cur = 0;
    cudaGetDevice(&cur);
    work(0);
    cudaSetDevice(cur);
  }
  for (auto& t : pool) t.join();
  for (int g = 0; g < ndev; ++g)
    if (rcs[g]) return fail(rcs[g], "shard %d (device %d): %s", g, devices[g], msgs[g].c_str());
  // words shared by two shards: each holds only its own windows' bits, so OR is the merge
  for (int g = 0; g < ndev; ++g)
    for (int k = 0; k < 2; ++k)
      if (edge_idx[2 * g + k] >= 0) bits_host[edge_idx[2 * g + k]] = 0;
  for (int g = 0; g < ndev; ++g)
    for (int k = 0; k < 2; ++k)
      if (edge_idx[2 * g + k] >= 0) bits_host[edge_idx[2 * g + k]] |= edges[2 * g + k];
  return VT_OK;
}

}  // extern "C"
