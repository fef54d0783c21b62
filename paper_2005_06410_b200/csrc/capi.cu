// capi.cu -- the C-ABI boundary (include/convgemm_b200.h): geometry validation with
// the reference's error semantics, operator/precision selection, device workspace
// accounting (the ScratchTracker equivalent) and kernel dispatch.
//
// Reference interfaces replaced (all under /root/reference/proj/include/convgemm/):
//   conv_gemm            conv.hpp:78-91     -> cgb_conv(CGB_ALGO_FUSED, ...)
//   conv_im2col_gemm     conv.hpp:60-74     -> cgb_conv(CGB_ALGO_EXPLICIT, ...)
//   im2col               im2col.hpp:77-120  -> cgb_im2col
//   output_dims/gemm_dims conv_params.hpp:27-43
//   ScratchTracker       scratch.hpp:14-28, src/scratch.cpp:12-52
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>
#include <string>
#include <type_traits>

#include "../../include/convgemm_b200.h"
#include "internal.h"

namespace cgb {

static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaError_t capture_safe_malloc(void** p, size_t bytes, bool zero) {
  cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
  cudaThreadExchangeStreamCaptureMode(&mode);
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess && zero) {
    static thread_local cudaStream_t side = nullptr;
    if (!side) e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(*p, 0, bytes, side);
    if (e == cudaSuccess) e = cudaStreamSynchronize(side);
  }
  cudaThreadExchangeStreamCaptureMode(&mode);
  if (e != cudaSuccess) cudaGetLastError();
  return e;
}

bool can_free_now(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs == cudaStreamCaptureStatusNone;
}

// ------------------------------------------------------------------ tuning
static std::mutex g_tune_mu;
static Tuning g_tune;

#define CGB_TUNING_KEYS(X)                                                                                   \
  X(sk) X(tail) X(pair) X(cfg) X(mt) X(bn) X(tma_a) X(tma_deep) X(pstore) X(pdl) X(verbose) X(smem_pad_kb) X(tps) X(splitk) X(k2_flo) X(b_res) X(urot) X(waste_pct) X(sk_pen_pct) X(strip_h) \
  X(host_chunk_kb) X(host_no_bounce) X(host_copy_threads) X(debug)

Tuning tuning() {
  Tuning t;
  {
    std::lock_guard<std::mutex> lk(g_tune_mu);
    t = g_tune;
  }
#ifdef CGB_PROFILING
  auto env = [](const char* k, auto& v) {
    if (const char* e = getenv(k)) v = (std::remove_reference_t<decltype(v)>)atoll(e);
  };
  env("CGB_SW_SK", t.sk); env("CGB_SW_TAIL", t.tail); env("CGB_SW_PAIR", t.pair); env("CGB_SW_CFG", t.cfg);
  env("CGB_SW_MT", t.mt); env("CGB_SW_BN", t.bn); env("CGB_SW_TMA_A", t.tma_a); env("CGB_SW_TMA_DEEP", t.tma_deep);
  env("CGB_SW_PSTORE", t.pstore); env("CGB_PDL", t.pdl); env("CGB_SW_VERBOSE", t.verbose);
  env("CGB_SW_SMEM_PAD", t.smem_pad_kb); env("CGB_HOST_CHUNK_KB", t.host_chunk_kb);
  env("CGB_HOST_NO_BOUNCE", t.host_no_bounce); env("CGB_HOST_COPY_THREADS", t.host_copy_threads);
  env("CGB_DEBUG_SW", t.debug); env("CGB_SW_TPS", t.tps); env("CGB_SW_SPLITK", t.splitk); env("CGB_K2_FLO", t.k2_flo); env("CGB_SW_BRES", t.b_res); env("CGB_SW_UROT", t.urot);
#endif
  return t;
}

static thread_local std::string g_last_error;
static thread_local int g_last_path = 0;

static cgb_status fail(cgb_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

static cgb_status cuda_fail(cudaError_t e, const char* where) {
  return fail(CGB_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ geometry (conv_params.hpp:27-43)
static cgb_status make_geom(const cgb_conv_params* cp, ConvGeom* g) {
  if (!cp) return fail(CGB_INVALID_ARGUMENT, "null ConvParams");
  if (cp->k_n < 1 || cp->k_h < 1 || cp->k_w < 1 || cp->c_i < 1 || cp->h_i < 1 || cp->w_i < 1 || cp->b < 1 ||
      cp->s < 1 || cp->p < 0)
    return fail(CGB_INVALID_GEOMETRY, "conv extents must be positive (padding non-negative)");
  const int64_t dh = cp->h_i - cp->k_h + 2 * cp->p;
  const int64_t dw = cp->w_i - cp->k_w + 2 * cp->p;
  if (dh < 0 || dw < 0) return fail(CGB_INVALID_GEOMETRY, "filter exceeds padded input");
  g->k_n = cp->k_n; g->k_h = cp->k_h; g->k_w = cp->k_w; g->c_i = cp->c_i;
  g->h_i = cp->h_i; g->w_i = cp->w_i; g->b = cp->b; g->s = cp->s; g->p = cp->p;
  g->h_o = dh / cp->s + 1;
  g->w_o = dw / cp->s + 1;
  g->m = cp->k_n;
  g->n = g->h_o * g->w_o * cp->b;
  g->k = cp->k_h * cp->k_w * cp->c_i;
  return CGB_OK;
}

// Index-width limits of the device kernels (32-bit per-image / per-row offsets).
static cgb_status check_device_limits(const ConvGeom& g) {
  const int64_t lim = (int64_t(1) << 31) - 1;
  if (g.c_i * g.h_i * g.w_i > lim || g.k > lim || g.h_o * g.w_o > lim || g.k_n > lim)
    return fail(CGB_UNSUPPORTED, "per-image extents exceed the 32-bit device indexing range");
  return CGB_OK;
}

// ------------------------------------------------------------------ TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

cudaError_t make_filter_tmap(CUtensorMap* tm, const float* f, int64_t k_n, int64_t K, int64_t ldf) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)k_n, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)(ldf * 4)};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(f), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_bhat_tmap(CUtensorMap* tm, const float* b, int64_t K, int64_t n, int64_t ldb) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)(ldb * 4)};
  cuuint32_t box[2] = {32, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(b), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_filter_tmap_tapmajor(CUtensorMap* tm, const float* f, const ConvGeom& g) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  const int64_t taps = g.k_h * g.k_w;
  cuuint64_t dims[3] = {(cuuint64_t)g.k_n, (cuuint64_t)taps, (cuuint64_t)g.c_i};
  cuuint64_t strides[2] = {(cuuint64_t)(g.k_n * 4), (cuuint64_t)(g.k_n * taps * 4)};
  cuuint32_t box[3] = {32, 1, 32};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(f), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_input_tmap_1x1(CUtensorMap* tm, const float* i, const ConvGeom& g) {
  auto enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  const int64_t hw = g.h_i * g.w_i;
  cuuint64_t dims[3] = {(cuuint64_t)hw, (cuuint64_t)g.c_i, (cuuint64_t)g.b};
  cuuint64_t strides[2] = {(cuuint64_t)(hw * 4), (cuuint64_t)(hw * g.c_i * 4)};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(i), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// ------------------------------------------------------------------ workspace (ScratchTracker)
// One cached device buffer per (device, stream): calls on different streams (which may
// run concurrently) never share workspace, like the stream-K counters. Accounting
// follows the reference's ScratchTracker (scratch.cpp:12-52): every call claims `need`
// bytes -- checked against the limit on EVERY call, cached buffer or not -- and
// current/peak count the claimed bytes of in-flight claims (released when the call has
// been enqueued), independent of the size of the cached allocation. A buffer that was
// in use while its stream was being captured into a CUDA graph may be referenced by
// that graph: it is never freed implicitly (retired to a list that only
// cgb_scratch_release frees; replaying graphs captured before a release is the
// caller's error, as freeing any buffer a graph uses).
struct WsBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  bool captured = false;  // used during a stream capture at least once
};
struct Scratch {
  std::mutex mu;
  std::map<std::pair<int, cudaStream_t>, WsBuf> bufs;
  std::vector<void*> retired;  // captured buffers that were outgrown
  std::atomic<uint64_t> current{0}, peak{0}, limit{0};
};
static Scratch g_scratch;

static void scratch_account(uint64_t need) {
  const uint64_t cur = g_scratch.current.fetch_add(need) + need;
  uint64_t seen = g_scratch.peak.load();
  while (seen < cur && !g_scratch.peak.compare_exchange_weak(seen, cur)) {
  }
}

// Claim `need` bytes of workspace for one call on stream st; the claim is released
// with scratch_done(need) once the call's kernels are enqueued.
static cgb_status scratch_get(size_t need, void** out, cudaStream_t st) {
  const uint64_t lim = g_scratch.limit.load();
  if (lim != 0 && need > lim)
    return fail(CGB_ALLOCATION_FAILURE, "workspace limit exceeded: " + std::to_string(need) +
                                            " bytes requested, limit " + std::to_string(lim));
  std::lock_guard<std::mutex> lk(g_scratch.mu);
  int dev = 0;
  cudaGetDevice(&dev);
  WsBuf& w = g_scratch.bufs[{dev, st}];
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) {
    cudaGetLastError();
    cs = cudaStreamCaptureStatusActive;  // unknown: treat as captured (never free)
  }
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  if (!w.ptr || w.bytes < need) {
    if (w.ptr) {
      // cudaFree synchronises the device, so no kernel still reads it -- unless a
      // captured graph refers to it: retire instead of freeing
      if (w.captured || capturing) g_scratch.retired.push_back(w.ptr);
      else cudaFree(w.ptr);
      w = WsBuf{};
    }
    void* p = nullptr;
    const size_t alloc = std::max<size_t>(need, size_t(1) << 20);
    if (capture_safe_malloc(&p, alloc) != cudaSuccess)
      return fail(CGB_ALLOCATION_FAILURE, "cannot allocate " + std::to_string(alloc) + " bytes of device workspace");
    w.ptr = p;
    w.bytes = alloc;
  }
  w.captured = w.captured || capturing;
  scratch_account(need);
  *out = w.ptr;
  return CGB_OK;
}

static void scratch_done(size_t need) { g_scratch.current.fetch_sub(need); }

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// Workspace plan for one call: filter copies (hi[, lo]) then B-hat.
struct Plan {
  int algo, prec;
  bool direct_filters;  // TF32 mode reading F itself through TMA (no filter workspace)
  int64_t ldf, ldb;
  int64_t f_bytes, b_bytes;
};

static bool tf32_family(int prec) { return prec == CGB_PREC_TF32 || prec == CGB_PREC_3XTF32; }

static int resolve_precision(int prec, const ConvGeom& g) {
  if (prec != CGB_PREC_AUTO) return prec;
  // fp32-accurate choice by measured cost: 3xTF32 on the tensor cores wherever a
  // shifted-window kernel takes the layer -- including the low-channel w-im2col rows
  // (VGG conv1, K = 27: 323 us vs 508 us for FFMA at b=64, profiles/r01_configs.json);
  // FFMA only for short contractions no tensor-core layout covers.
  if (g.k < 32 && !shifted_supported(g) && !wim_supported(g)) return CGB_PREC_FFMA;
  return CGB_PREC_3XTF32;
}

static bool use_wim(int algo, int prec, const ConvGeom& g) {
  return algo == CGB_ALGO_FUSED && tf32_family(prec) && !shifted_supported(g) && wim_supported(g);
}
static int64_t wim_filter_bytes(int prec, const ConvGeom& g) {
  return align_up(g.k_n * g.k_h * 32 * 4, 256) * (prec == CGB_PREC_3XTF32 ? 2 : 1);
}

static Plan make_plan(int algo, int prec, const ConvGeom& g, const float* F) {
  Plan pl{};
  pl.algo = algo;
  pl.prec = prec;
  pl.ldf = align_up(g.k_n, 4);
  // TF32 reads F itself through TMA. So does the explicit 3xTF32 path when the K2 kernel
  // splits the filter lo tile in shared memory (k2_gemm.cu): large static weights (fc
  // layers) then need no per-call split pass and no hi/lo workspace.
  const Tuning tu = tuning();
  const bool k2_flo = algo == CGB_ALGO_EXPLICIT && prec == CGB_PREC_3XTF32 &&
                      (tu.k2_flo > 0 || (tu.k2_flo == 0 && g.k_n * g.k * 4 > (int64_t(8) << 20)));
  pl.direct_filters = (prec == CGB_PREC_TF32 || k2_flo) && g.k_n % 4 == 0 &&
                      (F == nullptr || reinterpret_cast<uintptr_t>(F) % 16 == 0);
  if (tf32_family(prec) && !pl.direct_filters)
    pl.f_bytes = align_up(pl.ldf * g.k * 4, 256) * (prec == CGB_PREC_3XTF32 ? 2 : 1);
  pl.ldb = align_up(g.k, 4);
  if (algo == CGB_ALGO_EXPLICIT) pl.b_bytes = align_up(pl.ldb * g.n * 4, 256);
  return pl;
}

}  // namespace cgb

using namespace cgb;

extern "C" {

cgb_status cgb_output_dims(const cgb_conv_params* cp, int64_t* h_o, int64_t* w_o) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (h_o) *h_o = g.h_o;
  if (w_o) *w_o = g.w_o;
  return CGB_OK;
}

cgb_status cgb_gemm_dims(const cgb_conv_params* cp, int64_t* m, int64_t* n, int64_t* k) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (m) *m = g.m;
  if (n) *n = g.n;
  if (k) *k = g.k;
  return CGB_OK;
}

int64_t cgb_im2col_workspace_bytes(const cgb_conv_params* cp) {
  ConvGeom g;
  if (make_geom(cp, &g)) return -1;
  return g.k * g.n * (int64_t)sizeof(float);
}

cgb_status cgb_validate_blocking(const cgb_blocking_params* bp) {
  if (!bp) return CGB_OK;  // BlockingParams{} defaults are valid
  if (bp->mc < 1 || bp->nc < 1 || bp->kc < 1 || bp->mr < 1 || bp->nr < 1)
    return fail(CGB_INVALID_ARGUMENT, "blocking parameters must be positive");
  if (bp->mr > bp->mc || bp->nr > bp->nc)
    return fail(CGB_INVALID_ARGUMENT, "micro-tile must fit the cache block (mr<=mc, nr<=nc)");
  if (bp->mr * bp->nr > 4096) return fail(CGB_INVALID_ARGUMENT, "micro-tile mr*nr exceeds the supported maximum");
  return CGB_OK;
}

int64_t cgb_conv_workspace_bytes(int algo, int precision, const cgb_conv_params* cp) {
  ConvGeom g;
  if (make_geom(cp, &g)) return -1;
  if (algo == CGB_ALGO_DIRECT) return 0;
  const int prec = resolve_precision(precision, g);
  const Plan pl = make_plan(algo, prec, g, nullptr);
  return std::max<int64_t>(pl.f_bytes + pl.b_bytes, use_wim(algo, prec, g) ? wim_filter_bytes(prec, g) : 0);
}

int64_t cgb_gemm_workspace_bytes(int precision, int64_t m, int64_t n, int64_t k) {
  if (m < 1 || n < 1 || k < 1) return -1;
  cgb_conv_params cp{m, 1, 1, k, 1, 1, n, 1, 0};  // as cgb_gemm: a 1x1 conv over 1x1 images
  ConvGeom g;
  if (make_geom(&cp, &g)) return -1;
  return make_plan(CGB_ALGO_EXPLICIT, resolve_precision(precision, g), g, nullptr).f_bytes;  // B is the caller's
}

// The operator body behind cgb_conv and cgb_gemm. Bext != NULL: the lowered matrix B
// (k x n, leading dimension ldb_ext) is the caller's (gemm over a MatrixSource,
// gemm.hpp:100-105): the explicit path without the im2col step or its workspace.
static cgb_status conv_impl(int algo, int precision, const float* F, const float* I, const ConvGeom& g, float* O,
                            void* workspace, size_t workspace_bytes, void* stream, const float* Bext,
                            int64_t ldb_ext) {
  cgb_status st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (algo == CGB_ALGO_DIRECT) {  // the reference's seven-loop convolution (no workspace)
    const cudaError_t e = launch_direct_conv(F, I, O, g, s);
    if (e != cudaSuccess) return cuda_fail(e, "conv_direct kernel launch");
    g_last_path = 8;
    return CGB_OK;
  }
  const int prec = resolve_precision(precision, g);
  Plan pl = make_plan(algo, prec, g, F);
  if (Bext) {
    pl.b_bytes = 0;
    pl.ldb = ldb_ext;
  }
  // low-channel layers (c_i < 16: the stem, VGG conv1) on the tensor cores: w-im2col mode
  const bool wim = !Bext && use_wim(algo, prec, g);
  const size_t need = std::max<size_t>((size_t)(pl.f_bytes + pl.b_bytes), wim ? (size_t)wim_filter_bytes(prec, g) : 0);
  uint8_t* ws = nullptr;
  size_t claimed = 0;
  if (need > 0) {
    if (workspace) {
      if (workspace_bytes < need)
        return fail(CGB_ALLOCATION_FAILURE, "caller workspace too small: need " + std::to_string(need) + " bytes");
      ws = static_cast<uint8_t*>(workspace);
    } else {
      void* p = nullptr;
      if ((st = scratch_get(need, &p, s))) return st;
      ws = static_cast<uint8_t*>(p);
      claimed = need;
    }
  }
  struct Release {
    size_t n;
    ~Release() {
      if (n) scratch_done(n);
    }
  } release{claimed};
  cudaError_t e;
  // Filters for the tensor-core paths.
  const float* f_hi = F;
  const float* f_lo = nullptr;
  int64_t ldf = g.k_n;
  if (wim) {
    float* hi = reinterpret_cast<float*>(ws);
    float* lo = prec == CGB_PREC_3XTF32 ? reinterpret_cast<float*>(ws + wim_filter_bytes(prec, g) / 2) : nullptr;
    if ((e = launch_wim_filter_prep(F, hi, lo, g, s)) != cudaSuccess) return cuda_fail(e, "wim filter_prep");
    e = launch_tc_conv_wim(hi, lo, I, O, g, prec == CGB_PREC_3XTF32, s);
    if (e == cudaSuccess) {
      g_last_path = 7;
      return CGB_OK;
    }
    if (e != cudaErrorNotSupported) return cuda_fail(e, "conv kernel launch");
    // no fitting configuration: the generic kernels below (the workspace covers both)
  }
  if (tf32_family(prec)) {
    if (pl.direct_filters) {
      f_hi = F;
      ldf = g.k_n;
    } else {
      float* hi = reinterpret_cast<float*>(ws);
      float* lo = prec == CGB_PREC_3XTF32 ? reinterpret_cast<float*>(ws + pl.f_bytes / 2) : nullptr;
      if ((e = launch_filter_prep(F, hi, lo, pl.ldf, g, s)) != cudaSuccess) return cuda_fail(e, "filter_prep");
      f_hi = hi;
      f_lo = lo;
      ldf = pl.ldf;
    }
  }
  const float* Bhat = Bext;
  if (algo == CGB_ALGO_EXPLICIT && !Bext) {
    float* B = reinterpret_cast<float*>(ws + pl.f_bytes);
    if ((e = launch_im2col(I, B, pl.ldb, g, s)) != cudaSuccess) return cuda_fail(e, "im2col");
    Bhat = B;
  }
  if (prec == CGB_PREC_FFMA) {
    e = launch_ffma_conv(F, I, Bhat, pl.ldb, O, g, s);
    g_last_path = Bhat ? 4 : 3;
  } else {
    const bool split = prec == CGB_PREC_3XTF32;
    e = cudaErrorNotSupported;
    if (!Bhat && shifted_supported(g) && ldf == g.k_n) {
      e = launch_tc_conv_shifted(f_hi, f_lo, ldf, I, O, g, split, s);
      g_last_path = 5;
    }
    if (e != cudaErrorNotSupported) {
      // launched (or failed for real)
    } else if (!Bhat && gather_supported(g) && ldf == g.k_n) {
      e = launch_tc_gather(f_hi, f_lo, I, O, g, split, s);
      g_last_path = 6;
    } else if (Bhat) {  // explicit path: TMA-fed GEMM over the lowered matrix (K2)
      e = launch_k2_gemm(f_hi, f_lo, ldf, Bhat, pl.ldb, O, g, split, s);
      g_last_path = 2;
    } else {
      e = launch_tc_conv(f_hi, f_lo, ldf, I, O, g, split, s);
      g_last_path = 1;
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "conv kernel launch");
  return CGB_OK;
}

cgb_status cgb_conv(int algo, int precision, const float* F, const float* I, const cgb_conv_params* cp, float* O,
                    void* workspace, size_t workspace_bytes, void* stream) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (algo != CGB_ALGO_EXPLICIT && algo != CGB_ALGO_FUSED && algo != CGB_ALGO_DIRECT)
    return fail(CGB_INVALID_ARGUMENT, "unknown algo");
  if (precision < CGB_PREC_AUTO || precision > CGB_PREC_FFMA)
    return fail(CGB_INVALID_ARGUMENT, "unknown precision");
  if (!F || !I || !O) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  if ((st = check_device_limits(g))) return st;
  return conv_impl(algo, precision, F, I, g, O, workspace, workspace_bytes, stream, nullptr, 0);
}

// C (m x n) = A (m x k) * B (k x n), column-major: a 1x1 convolution over 1x1 images
// (F = A as k_n=m x c_i=k, I = B as c_i=k x b=n, O = C), run as the explicit path
// with B itself as the lowered matrix (the reference's fc layers, bench.cpp:140-153).
cgb_status cgb_gemm(int precision, const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                    int64_t m, int64_t n, int64_t k, void* workspace, size_t workspace_bytes, void* stream) {
  if (m < 1 || n < 1 || k < 1) return fail(CGB_INVALID_GEOMETRY, "gemm dimensions must be positive");
  if (lda != m || ldc != m || ldb < k)
    return fail(CGB_DIMENSION_MISMATCH, "gemm needs lda == m, ldc == m and ldb >= k (dense column-major A and C)");
  if (precision < CGB_PREC_AUTO || precision > CGB_PREC_FFMA)
    return fail(CGB_INVALID_ARGUMENT, "unknown precision");
  if (!A || !B || !C) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  cgb_conv_params cp{m, 1, 1, k, 1, 1, n, 1, 0};
  ConvGeom g;
  cgb_status st = make_geom(&cp, &g);
  if (st) return st;
  if ((st = check_device_limits(g))) return st;
  // The explicit-path kernels read B in 16-byte vectors: an unaligned B (or ld) is
  // lowered into an aligned, zero-padded copy first (im2col of a 1x1 conv is exactly that).
  if (ldb % 4 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0)
    return conv_impl(CGB_ALGO_EXPLICIT, precision, A, B, g, C, workspace, workspace_bytes, stream, B, ldb);
  if (ldb != k) return fail(CGB_DIMENSION_MISMATCH, "gemm needs ldb == k or a multiple of 4 (16-byte aligned B)");
  return conv_impl(CGB_ALGO_EXPLICIT, precision, A, B, g, C, workspace, workspace_bytes, stream, nullptr, 0);
}

cgb_status cgb_conv_gemm(const float* F, const float* I, const cgb_conv_params* cp, const cgb_blocking_params* bp,
                         int threads, float* O, int precision, void* stream) {
  (void)threads;
  cgb_status st = cgb_validate_blocking(bp);
  if (st) return st;
  return cgb_conv(CGB_ALGO_FUSED, precision, F, I, cp, O, nullptr, 0, stream);
}

cgb_status cgb_conv_im2col_gemm(const float* F, const float* I, const cgb_conv_params* cp,
                                const cgb_blocking_params* bp, int threads, float* O, int precision, void* stream) {
  (void)threads;
  cgb_status st = cgb_validate_blocking(bp);
  if (st) return st;
  return cgb_conv(CGB_ALGO_EXPLICIT, precision, F, I, cp, O, nullptr, 0, stream);
}

cgb_status cgb_im2col(const float* I, const cgb_conv_params* cp, float* B, int64_t ldb, void* stream) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (!I || !B) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  if (ldb < g.k) return fail(CGB_DIMENSION_MISMATCH, "leading dimension smaller than k");
  if ((st = check_device_limits(g))) return st;
  cudaError_t e = launch_im2col(I, B, ldb, g, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "im2col");
  return CGB_OK;
}

// Host-memory entry point with the reference's synchronous semantics.
cgb_status cgb_conv_host(int algo, int precision, const float* F_host, const float* I_host,
                         const cgb_conv_params* cp, float* O_host, void* stream) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (!F_host || !I_host || !O_host) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t fb = (size_t)(g.k_n * g.k) * 4, ib = (size_t)(g.c_i * g.h_i * g.w_i * g.b) * 4,
               ob = (size_t)(g.k_n * g.n) * 4;
  // Device staging buffers for the host path, cached across calls (not workspace).
  static std::mutex mu;
  static void* buf = nullptr;
  static size_t cap = 0;
  static int dev_of_buf = -1;
  std::lock_guard<std::mutex> lk(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t need = (size_t)align_up((int64_t)fb, 256) + (size_t)align_up((int64_t)ib, 256) + ob;
  if (!buf || cap < need || dev_of_buf != dev) {
    if (buf) cudaFree(buf);
    buf = nullptr;
    if (cudaMalloc(&buf, need) != cudaSuccess) {
      cudaGetLastError();
      cap = 0;
      return fail(CGB_ALLOCATION_FAILURE, "cannot allocate device staging for the host path");
    }
    cap = need;
    dev_of_buf = dev;
  }
  uint8_t* b = static_cast<uint8_t*>(buf);
  float* dF = reinterpret_cast<float*>(b);
  float* dI = reinterpret_cast<float*>(b + align_up((int64_t)fb, 256));
  float* dO = reinterpret_cast<float*>(b + align_up((int64_t)fb, 256) + align_up((int64_t)ib, 256));
  // Batch-chunked pipeline (host_pipe.cu): image i of I and of O are contiguous byte
  // ranges, so chunk [i0, i0+n) is a conv with b = n on offset pointers.
  struct Ctx {
    int algo, precision;
    const float* dF;
    const float* dI;
    float* dO;
    cgb_conv_params cp;
    size_t in_items, out_items;
    cgb_status st;
  } ctx{algo, precision, dF, dI, dO, *cp, ib / 4 / (size_t)g.b, ob / 4 / (size_t)g.b, CGB_OK};
  HostPipe io;
  io.extra.push_back({dF, F_host, fb});
  io.in_host = I_host;
  io.in_dev = dI;
  io.in_item = ib / (size_t)g.b;
  io.out_host = O_host;
  io.out_dev = dO;
  io.out_item = ob / (size_t)g.b;
  io.items = g.b;
  io.chunk_items = host_chunk_items(io.in_item, io.out_item, g.b);
  io.ctx = &ctx;
  io.compute = [](void* p, int64_t i0, int64_t n, cudaStream_t st) -> cudaError_t {
    Ctx& c = *static_cast<Ctx*>(p);
    cgb_conv_params q = c.cp;
    q.b = n;
    c.st = cgb_conv(c.algo, c.precision, c.dF, c.dI + (size_t)i0 * c.in_items, &q, c.dO + (size_t)i0 * c.out_items,
                    nullptr, 0, st);
    return c.st == CGB_OK ? cudaSuccess : cudaErrorUnknown;
  };
  std::string where;
  const cudaError_t e = run_host_pipeline(io, s, &where);
  if (ctx.st != CGB_OK) return ctx.st;  // cgb_conv already set the message
  if (e != cudaSuccess) return cuda_fail(e, where.c_str());
  return CGB_OK;
}

// ---- host-pointer im2col and gemm (the reference's other host entry points)
namespace {
struct DevBuf {  // device staging for one synchronous host call
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc(&p, std::max<size_t>(n, 256)); }
};
}  // namespace

cgb_status cgb_im2col_host(const float* I_host, const cgb_conv_params* cp, float* B_host, int64_t ldb) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (!I_host || !B_host) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  if (ldb < g.k) return fail(CGB_DIMENSION_MISMATCH, "leading dimension smaller than k");
  if ((st = check_device_limits(g))) return st;
  const size_t ib = (size_t)(g.h_i * g.w_i * g.c_i * g.b) * 4, bb = (size_t)(ldb * g.n) * 4;
  DevBuf dI, dB;
  cudaError_t e;
  if ((e = dI.alloc(ib)) != cudaSuccess || (e = dB.alloc(bb)) != cudaSuccess) {
    cudaGetLastError();
    return fail(CGB_ALLOCATION_FAILURE, "cannot allocate device staging for im2col");
  }
  if ((e = cudaMemcpy(dI.p, I_host, ib, cudaMemcpyHostToDevice)) != cudaSuccess) return cuda_fail(e, "im2col H2D");
  if ((e = launch_im2col(static_cast<const float*>(dI.p), static_cast<float*>(dB.p), ldb, g, nullptr)) != cudaSuccess)
    return cuda_fail(e, "im2col");
  if ((e = cudaMemcpy(B_host, dB.p, bb, cudaMemcpyDeviceToHost)) != cudaSuccess) return cuda_fail(e, "im2col D2H");
  return CGB_OK;
}

cgb_status cgb_gemm_host(int precision, const float* A_host, int64_t lda, const float* B_host, int64_t ldb,
                         float* C_host, int64_t ldc, int64_t m, int64_t n, int64_t k, int accumulate) {
  if (m < 1 || n < 1 || k < 1) return fail(CGB_INVALID_GEOMETRY, "gemm dimensions must be positive");
  if (lda < m || ldb < k || ldc < m) return fail(CGB_DIMENSION_MISMATCH, "leading dimension smaller than rows");
  if (!A_host || !B_host || !C_host) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  const int64_t ldbp = (k + 3) / 4 * 4;  // the device B gets a 16-byte leading dimension
  DevBuf dA, dB, dC;
  cudaError_t e;
  if ((e = dA.alloc((size_t)(m * k) * 4)) != cudaSuccess || (e = dB.alloc((size_t)(ldbp * n) * 4)) != cudaSuccess ||
      (e = dC.alloc((size_t)(m * n) * 4)) != cudaSuccess) {
    cudaGetLastError();
    return fail(CGB_ALLOCATION_FAILURE, "cannot allocate device staging for gemm");
  }
  // dense copies (the device kernels take lda == ldc == m)
  if ((e = cudaMemcpy2D(dA.p, (size_t)m * 4, A_host, (size_t)lda * 4, (size_t)m * 4, (size_t)k,
                        cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy2D(dB.p, (size_t)ldbp * 4, B_host, (size_t)ldb * 4, (size_t)k * 4, (size_t)n,
                        cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "gemm H2D");
  if (ldbp != k && (e = cudaMemset2D(static_cast<char*>(dB.p) + k * 4, (size_t)ldbp * 4, 0, (size_t)(ldbp - k) * 4,
                                     (size_t)n)) != cudaSuccess)
    return cuda_fail(e, "gemm B padding");
  cgb_status st = cgb_gemm(precision, static_cast<const float*>(dA.p), m, static_cast<const float*>(dB.p), ldbp,
                           static_cast<float*>(dC.p), m, m, n, k, nullptr, 0, nullptr);
  if (st) return st;
  std::vector<float> tmp;
  float* dst = C_host;
  int64_t ldd = ldc;
  if (accumulate) {
    tmp.resize((size_t)(m * n));
    dst = tmp.data();
    ldd = m;
  }
  if ((e = cudaMemcpy2D(dst, (size_t)ldd * 4, dC.p, (size_t)m * 4, (size_t)m * 4, (size_t)n,
                        cudaMemcpyDeviceToHost)) != cudaSuccess)
    return cuda_fail(e, "gemm D2H");
  if (accumulate)
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < m; ++i) C_host[i + j * ldc] += tmp[(size_t)(i + j * m)];
  return CGB_OK;
}

// ---- float64: the reference's f64 instantiations on the device, bit-identical
static int64_t kc_of(const cgb_blocking_params* bp) { return bp ? bp->kc : 640; }

cgb_status cgb_conv_f64(int algo, const double* F, const double* I, const cgb_conv_params* cp,
                        const cgb_blocking_params* bp, double* O, void* stream) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if ((st = cgb_validate_blocking(bp))) return st;
  if (!F || !I || !O) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  if (algo != CGB_ALGO_EXPLICIT && algo != CGB_ALGO_FUSED && algo != CGB_ALGO_DIRECT)
    return fail(CGB_INVALID_ARGUMENT, "unknown algo");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (algo == CGB_ALGO_DIRECT) {
    e = launch_direct_conv_f64(F, I, O, g, s);
  } else if (algo == CGB_ALGO_FUSED) {
    e = launch_refgemm_f64(F, g.k_n, nullptr, 0, I, g, O, g.k_n, g.m, g.n, g.k, kc_of(bp), false, s);
  } else {
    // the reference materialises B-hat (k x n) and runs the same gemm over it
    void* ws = nullptr;
    const size_t need = (size_t)(g.k * g.n) * sizeof(double);
    if ((st = scratch_get(need, &ws, s))) return st;
    struct Release {
      size_t n;
      ~Release() { scratch_done(n); }
    } release{need};
    double* B = static_cast<double*>(ws);
    if ((e = launch_im2col_f64(I, B, g.k, g, s)) != cudaSuccess) return cuda_fail(e, "im2col f64");
    e = launch_refgemm_f64(F, g.k_n, B, g.k, nullptr, g, O, g.k_n, g.m, g.n, g.k, kc_of(bp), false, s);
  }
  if (e != cudaSuccess) return cuda_fail(e, "f64 conv kernel launch");
  g_last_path = 9;
  return CGB_OK;
}

cgb_status cgb_conv_host_f64(int algo, const double* F_host, const double* I_host, const cgb_conv_params* cp,
                             const cgb_blocking_params* bp, double* O_host) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (!F_host || !I_host || !O_host) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  const size_t fb = (size_t)(g.k_n * g.k) * 8, ib = (size_t)(g.c_i * g.h_i * g.w_i * g.b) * 8,
               ob = (size_t)(g.k_n * g.n) * 8;
  DevBuf dF, dI, dO;
  cudaError_t e;
  if ((e = dF.alloc(fb)) != cudaSuccess || (e = dI.alloc(ib)) != cudaSuccess || (e = dO.alloc(ob)) != cudaSuccess) {
    cudaGetLastError();
    return fail(CGB_ALLOCATION_FAILURE, "cannot allocate device staging for the f64 host path");
  }
  if ((e = cudaMemcpy(dF.p, F_host, fb, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dI.p, I_host, ib, cudaMemcpyHostToDevice)) != cudaSuccess)
    return cuda_fail(e, "f64 H2D");
  if ((st = cgb_conv_f64(algo, static_cast<const double*>(dF.p), static_cast<const double*>(dI.p), cp, bp,
                         static_cast<double*>(dO.p), nullptr)))
    return st;
  if ((e = cudaMemcpy(O_host, dO.p, ob, cudaMemcpyDeviceToHost)) != cudaSuccess) return cuda_fail(e, "f64 D2H");
  return CGB_OK;
}

cgb_status cgb_im2col_host_f64(const double* I_host, const cgb_conv_params* cp, double* B_host, int64_t ldb) {
  ConvGeom g;
  cgb_status st = make_geom(cp, &g);
  if (st) return st;
  if (!I_host || !B_host) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  if (ldb < g.k) return fail(CGB_DIMENSION_MISMATCH, "leading dimension smaller than k");
  const size_t ib = (size_t)(g.h_i * g.w_i * g.c_i * g.b) * 8, bb = (size_t)(ldb * g.n) * 8;
  DevBuf dI, dB;
  cudaError_t e;
  if ((e = dI.alloc(ib)) != cudaSuccess || (e = dB.alloc(bb)) != cudaSuccess) {
    cudaGetLastError();
    return fail(CGB_ALLOCATION_FAILURE, "cannot allocate device staging for im2col");
  }
  if ((e = cudaMemcpy(dI.p, I_host, ib, cudaMemcpyHostToDevice)) != cudaSuccess) return cuda_fail(e, "im2col H2D");
  if ((e = launch_im2col_f64(static_cast<const double*>(dI.p), static_cast<double*>(dB.p), ldb, g, nullptr)) !=
      cudaSuccess)
    return cuda_fail(e, "im2col f64");
  if ((e = cudaMemcpy(B_host, dB.p, bb, cudaMemcpyDeviceToHost)) != cudaSuccess) return cuda_fail(e, "im2col D2H");
  return CGB_OK;
}

cgb_status cgb_gemm_host_f64(const double* A_host, int64_t lda, const double* B_host, int64_t ldb, double* C_host,
                             int64_t ldc, int64_t m, int64_t n, int64_t k, const cgb_blocking_params* bp,
                             int accumulate) {
  if (m < 1 || n < 1 || k < 1) return fail(CGB_INVALID_GEOMETRY, "gemm dimensions must be positive");
  if (lda < m || ldb < k || ldc < m) return fail(CGB_DIMENSION_MISMATCH, "leading dimension smaller than rows");
  if (!A_host || !B_host || !C_host) return fail(CGB_INVALID_ARGUMENT, "null tensor pointer");
  cgb_status st = cgb_validate_blocking(bp);
  if (st) return st;
  DevBuf dA, dB, dC;
  cudaError_t e;
  if ((e = dA.alloc((size_t)(lda * k) * 8)) != cudaSuccess || (e = dB.alloc((size_t)(ldb * n) * 8)) != cudaSuccess ||
      (e = dC.alloc((size_t)(ldc * n) * 8)) != cudaSuccess) {
    cudaGetLastError();
    return fail(CGB_ALLOCATION_FAILURE, "cannot allocate device staging for gemm");
  }
  if ((e = cudaMemcpy(dA.p, A_host, (size_t)(lda * k) * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (e = cudaMemcpy(dB.p, B_host, (size_t)(ldb * n) * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
      (accumulate && (e = cudaMemcpy(dC.p, C_host, (size_t)(ldc * n) * 8, cudaMemcpyHostToDevice)) != cudaSuccess))
    return cuda_fail(e, "gemm H2D");
  ConvGeom g{};
  if ((e = launch_refgemm_f64(static_cast<const double*>(dA.p), lda, static_cast<const double*>(dB.p), ldb, nullptr, g,
                              static_cast<double*>(dC.p), ldc, m, n, k, kc_of(bp), accumulate != 0, nullptr)) !=
      cudaSuccess)
    return cuda_fail(e, "gemm f64");
  if ((e = cudaMemcpy2D(C_host, (size_t)ldc * 8, dC.p, (size_t)ldc * 8, (size_t)m * 8, (size_t)n,
                        cudaMemcpyDeviceToHost)) != cudaSuccess)
    return cuda_fail(e, "gemm D2H");
  return CGB_OK;
}

uint64_t cgb_scratch_current_bytes(void) { return g_scratch.current.load(); }
uint64_t cgb_scratch_peak_bytes(void) { return g_scratch.peak.load(); }
void cgb_scratch_reset_peak(void) { g_scratch.peak.store(g_scratch.current.load()); }
void cgb_scratch_set_limit(uint64_t bytes) { g_scratch.limit.store(bytes); }
void cgb_scratch_release(void) {
  // frees every cached workspace, captured or not: graphs captured before this call must
  // not be replayed afterwards
  std::lock_guard<std::mutex> lk(g_scratch.mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& kv : g_scratch.bufs)
    if (kv.second.ptr) {
      cudaSetDevice(kv.first.first);
      cudaFree(kv.second.ptr);
    }
  for (void* p : g_scratch.retired) cudaFree(p);
  cudaSetDevice(cur);
  g_scratch.bufs.clear();
  g_scratch.retired.clear();
}
uint64_t cgb_scratch_cached_bytes(void) {
  std::lock_guard<std::mutex> lk(g_scratch.mu);
  uint64_t n = 0;
  for (auto& kv : g_scratch.bufs) n += kv.second.bytes;
  return n;
}

cgb_status cgb_set_tuning(const char* key, int64_t value) {
  if (!key) return fail(CGB_INVALID_ARGUMENT, "null tuning key");
  std::lock_guard<std::mutex> lk(g_tune_mu);
#define CGB_SET(k)                                  \
  if (strcmp(key, #k) == 0) {                       \
    g_tune.k = (decltype(g_tune.k))value;           \
    return CGB_OK;                                  \
  }
  CGB_TUNING_KEYS(CGB_SET)
#undef CGB_SET
  return fail(CGB_INVALID_ARGUMENT, std::string("unknown tuning key: ") + key);
}

cgb_status cgb_get_tuning(const char* key, int64_t* value) {
  if (!key || !value) return fail(CGB_INVALID_ARGUMENT, "null tuning key or output");
  const Tuning t = tuning();
#define CGB_GET(k)                    \
  if (strcmp(key, #k) == 0) {         \
    *value = (int64_t)t.k;            \
    return CGB_OK;                    \
  }
  CGB_TUNING_KEYS(CGB_GET)
#undef CGB_GET
  return fail(CGB_INVALID_ARGUMENT, std::string("unknown tuning key: ") + key);
}

const char* cgb_last_error(void) { return g_last_error.c_str(); }
const char* cgb_version(void) { return "convgemm-b200 0.1 (sm_100a)"; }
uint64_t cgb_kernel_launch_count(void) { return g_launches.load(); }
int cgb_last_path(void) { return g_last_path; }

}  // extern "C"
