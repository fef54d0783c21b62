// internal.h -- host-side interfaces between the C-ABI layer (capi.cu) and the
// kernel translation units. Not installed; no torch types.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "common.cuh"

namespace cgb {

// Dispatch-policy knobs. Every setting is correct: they only choose among equivalent
// kernel variants (tests force the rarer ones; tools sweep them). Set through
// cgb_set_tuning(); the product library reads no environment variables. Profiling builds
// (-DCGB_PROFILING, tools/) also take the CGB_* environment variables, read at every
// launch, plus the correctness-breaking CGB_DEBUG_SW stage switches.
struct Tuning {
  int sk = 1;            // stream-K split of the last rounds: 0 never, 1 by fill (3x3-like layers), 2 whenever it fits, 3 by fill incl. 1x1
  int tail = 1;          // tail tiles: 0 never, 1 by cost, 2 whenever they fit
  int pair = 1;          // CTA pairs (cta_group::2): 0 never, 1 by policy, 2 also for the w-im2col layers
  int cfg = -1;          // force one shifted-window candidate (index into kCands)
  int mt = 0;            // force the M tile (subtiles of 128 rows)
  int bn = 0;            // force the filter tile (64, 128, 256)
  int tma_a = 1;         // TMA-fed A for 1x1 stride-1 layers
  int tma_deep = 1;      // deep A rings for 1x1 layers
  int pstore = 1;        // lane-pair epilogue stores
  int pdl = 1;           // programmatic dependent launch
  int verbose = 0;       // print the chosen configuration to stderr
  int smem_pad_kb = 0;   // pad dynamic shared memory (shrinks the L1 carve-out)
  int tps = 0;           // shifted-window filter taps per stage hand-over (0 = by cost)
  int splitk = 0;        // split-K pieces for few-tile layers: -1 never, 0 auto, S forced
  int b_res = 1;         // shifted-window: keep the filters resident in the ring when they fit (0 = always stream)
  int urot = 1;          // shifted-window: rotate the window unit -> staging warp assignment per chunk
  int sk_pen_pct = 130;  // M-tile cost model: cost factor (percent) of a stream-K split that reaches every tile
                         // (fewer than two rounds) for filter tiles <= 128; 100 = the round-2 model
  int strip_h = 0;       // shifted window: h-strips of this many output rows for wide stride-1 images (0 = by rule, -1 = off)
  int waste_pct = 0;     // shifted-window domain: cap on padded-plane rows per real output row, in percent (0 = none)
  int k2_flo = 0;        // explicit 3xTF32: filter lo tile split in the kernel: -1 never, 0 by size, 1 always
  int64_t host_chunk_kb = 8192;  // host path: chunk size of the H2D || conv || D2H pipeline
  int host_no_bounce = 0;        // host path: DMA pageable buffers directly (no pinned ring)
  int host_copy_threads = 0;     // host path: memcpy pool size (0 = min(8, cores/2))
  int debug = 0;         // CGB_DEBUG_SW stage switches (profiling builds only)
};
// Snapshot of the current settings (profiling builds: overlaid with the environment).
Tuning tuning();

// Launch accounting (cgb_kernel_launch_count): every kernel launch site bumps it.
void count_launch(uint64_t n = 1);

// Device allocation that is legal while a stream is being captured into a CUDA graph
// (the thread's capture mode is relaxed around cudaMalloc; nothing is enqueued), and
// zero-filled when zero = true (on a private stream, synchronously).
cudaError_t capture_safe_malloc(void** p, size_t bytes, bool zero = false);
// True when the calling thread may free device memory now (no capture in progress on
// `st`; cudaFree would otherwise invalidate the capture).
bool can_free_now(cudaStream_t st);

// K1: explicit lowered matrix B (k x n, column-major, ld = ldb >= k), bit-exact
// with im2col<float> (im2col.hpp:77-120); rows k..ldb-1 zero-filled.
cudaError_t launch_im2col(const float* I, float* B, int64_t ldb, const ConvGeom& g, cudaStream_t st);

// K4: fp32 FFMA convolution on CUDA cores. explicit_src != nullptr selects the
// explicit path (A operand read from B with leading dimension ldb).
cudaError_t launch_ffma_conv(const float* F, const float* I, const float* explicit_src, int64_t ldb, float* O,
                             const ConvGeom& g, cudaStream_t st);

// The reference's arithmetic bit for bit (ref_order.cu): conv_direct (conv.hpp:24-55),
// the kc-blocked gemm order (gemm.hpp:46-97) and im2col, for float and double.
cudaError_t launch_direct_conv(const float* F, const float* I, float* O, const ConvGeom& g, cudaStream_t st);
cudaError_t launch_direct_conv_f64(const double* F, const double* I, double* O, const ConvGeom& g, cudaStream_t st);
// C = A * B in the reference's kc-blocked order; B == nullptr: the lowered matrix of g from I.
cudaError_t launch_refgemm_f64(const double* A, int64_t lda, const double* B, int64_t ldb, const double* I,
                               const ConvGeom& g, double* C, int64_t ldc, int64_t m, int64_t n, int64_t K, int64_t kc,
                               bool accumulate, cudaStream_t st);
cudaError_t launch_im2col_f64(const double* I, double* B, int64_t ldb, const ConvGeom& g, cudaStream_t st);

// K5: filter preparation. Writes F (k_n x K, ld = k_n) into hi (and lo when
// lo != nullptr) with leading dimension ldf >= k_n, zero padding n >= k_n.
// hi = tf32_rna(f), lo = tf32_rna(f - hi)  (3xTF32 split); with lo == nullptr hi = f.
cudaError_t launch_filter_prep(const float* F, float* hi, float* lo, int64_t ldf, const ConvGeom& g,
                               cudaStream_t st);

// K3: tcgen05 kind::tf32 implicit GEMM in the reference's row order (any geometry).
// Filters are read by TMA from (f_hi, f_lo) with leading dimension ldf (ldf*4 % 16 == 0).
cudaError_t launch_tc_conv(const float* f_hi, const float* f_lo, int64_t ldf, const float* I, float* O,
                           const ConvGeom& g, bool split, cudaStream_t st);

// K2 (k2_gemm.cu): the explicit path's GEMM over a lowered matrix Bhat (k x n, K-fastest,
// ld = ldb with ldb % 4 == 0, 16-byte aligned), both operands TMA-fed. f_lo == nullptr
// with split: the filter lo tile is computed in the kernel from the raw filters.
cudaError_t launch_k2_gemm(const float* f_hi, const float* f_lo, int64_t ldf, const float* Bhat, int64_t ldb,
                           float* O, const ConvGeom& g, bool split, cudaStream_t st);
// 2-D TMA descriptor over Bhat (K x n, ld = ldb floats): box 32 rows of K x 128 columns,
// 128-byte swizzle (the K-major UMMA A layout), out-of-range rows/columns read as zero.
cudaError_t make_bhat_tmap(CUtensorMap* tm, const float* b, int64_t K, int64_t n, int64_t ldb);
// Per-(device, stream) arrival counters (n ints, zero between launches) and partial-tile
// workspace for split launches (shifted_conv.cu); false when the allocation fails.
namespace sw {
bool sk_buffers(cudaStream_t st, size_t n, size_t ws_bytes, int** counters, float** ws);
}

// 2-D TMA descriptor over a filter matrix (k_n x K, leading dimension ldf floats):
// box 32 filters x 32 rows, 128-byte swizzle with 32-byte atoms (the MN-major
// kind::tf32 UMMA B layout, SWIZZLE_128B_BASE32B).
cudaError_t make_filter_tmap(CUtensorMap* tm, const float* f, int64_t k_n, int64_t K, int64_t ldf);

// 3-D TMA descriptor over F seen as (k_n, tap = i_kh + i_kw*k_h, c_i): box 32 filters x
// 1 tap x 32 channels, 32-byte-atom 128B swizzle. Needs k_n % 4 == 0.
cudaError_t make_filter_tmap_tapmajor(CUtensorMap* tm, const float* f, const ConvGeom& g);
// I viewed as (h*w pixels, c_i, b) with 32 x 32 x 1 boxes, SW128 32-byte atoms (1x1 layers)
cudaError_t make_input_tmap_1x1(CUtensorMap* tm, const float* i, const ConvGeom& g);

// K3 tap-major gather kernel (tc_gather.cu): c_i >= 16, k_n % 4 == 0.
bool gather_supported(const ConvGeom& g);
cudaError_t launch_tc_gather(const float* f_hi, const float* f_lo, const float* I, float* O, const ConvGeom& g,
                             bool split, cudaStream_t st);

// V2: stride/phase "shifted window" tcgen05 kernel; returns cudaErrorNotSupported
// when the geometry is outside its domain (caller falls back to launch_tc_conv).
bool shifted_supported(const ConvGeom& g);
// Low-channel mode of the shifted-window kernel ("w-im2col"): each window row holds the
// k_w*c_i values of one output row's w-taps (k_w*c_i <= 32), only the k_h taps are row
// shifts. For the stem and VGG conv1 (c_i = 3). Filters from launch_wim_filter_prep.
bool wim_supported(const ConvGeom& g);
cudaError_t launch_wim_filter_prep(const float* F, float* hi, float* lo, const ConvGeom& g, cudaStream_t st);
cudaError_t launch_tc_conv_wim(const float* f_hi, const float* f_lo, const float* I, float* O, const ConvGeom& g,
                               bool split, cudaStream_t st);
cudaError_t launch_tc_conv_shifted(const float* f_hi, const float* f_lo, int64_t ldf, const float* I, float* O,
                                   const ConvGeom& g, bool split, cudaStream_t st);

// Host-memory runtime (host_pipe.cu): batch-chunked H2D || compute || D2H over three
// streams, pinned bounce ring + parallel memcpy for pageable caller buffers.
struct HostPipe {
  struct Extra { void* dev; const void* host; size_t bytes; };
  std::vector<Extra> extra;  // copied H2D once, before the first chunk
  const void* in_host = nullptr;
  void* in_dev = nullptr;
  size_t in_item = 0;  // bytes per batch item (image) of the input
  void* out_host = nullptr;
  const void* out_dev = nullptr;
  size_t out_item = 0;
  int64_t items = 0, chunk_items = 0;
  // runs the device work for items [i0, i0+n) on st
  cudaError_t (*compute)(void* ctx, int64_t i0, int64_t n, cudaStream_t st) = nullptr;
  void* ctx = nullptr;
};
int64_t host_chunk_items(size_t in_item, size_t out_item, int64_t items);
cudaError_t run_host_pipeline(const HostPipe& io, cudaStream_t compute, std::string* where);

}  // namespace cgb
