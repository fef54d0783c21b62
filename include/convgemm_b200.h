/*
 * convgemm_b200.h -- C-ABI drop-in boundary of the B200-native convolution operator.
 *
 * Replaces the reference's header-only C++ conv API (/root/reference/proj/include/convgemm/):
 *
 *   cgb_conv_gemm           <- convgemm::conv_gemm<float>        conv.hpp:78-91  (fused: im2col inside B packing)
 *   cgb_conv_im2col_gemm    <- convgemm::conv_im2col_gemm<float> conv.hpp:60-74  (explicit: im2col, then gemm)
 *   cgb_conv                <- both of the above, plus the precision selector the B200 path adds
 *   cgb_im2col              <- convgemm::im2col<float>           im2col.hpp:77-120 (explicit lowered matrix)
 *   cgb_gemm                <- convgemm::gemm<float> over a MatrixSource gemm.hpp:46-105 (fc layers, bench.cpp:140-153)
 *   cgb_output_dims         <- convgemm::output_dims             conv_params.hpp:27-36
 *   cgb_gemm_dims           <- convgemm::gemm_dims               conv_params.hpp:40-43
 *   cgb_im2col_workspace_bytes <- convgemm::im2col_workspace_bytes im2col.hpp:36-39
 *   cgb_validate_blocking   <- convgemm::validate(BlockingParams) blocking.hpp:22-29
 *   cgb_scratch_*           <- convgemm::ScratchTracker          scratch.hpp:14-28, src/scratch.cpp:12-52
 *   cgb_conv_host           <- the synchronous host-memory semantics of the reference entry points
 *
 * Layouts are the reference's leftmost-fastest ones (tensor.hpp:28-50):
 *   F: k_n x k_h x k_w x c_i   I: h_i x w_i x c_i x b   O: k_n x h_o x w_o x b
 * Stride and symmetric zero padding are virtual (im2col.hpp:71-76). O is fully
 * overwritten (conv.hpp:71,89: zero_matrix then C += A*B).
 *
 * Device entry points take device pointers and an opaque stream handle
 * (a cudaStream_t; NULL = legacy default stream) and are asynchronous.
 * Errors are returned as cgb_status codes mirroring the reference's exception
 * types (types.hpp:15-41, blocking.hpp:22-29); cgb_last_error() returns the
 * message of the last failure on the calling thread.
 *
 * No torch or CUDA types appear in this header: plain pointers, sizes and PODs.
 */
#ifndef CONVGEMM_B200_H
#define CONVGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ConvParams, conv_params.hpp:8-16 (same field order, int64 = index_t). */
typedef struct cgb_conv_params {
    int64_t k_n, k_h, k_w, c_i, h_i, w_i, b, s, p;
} cgb_conv_params;

/* BlockingParams, blocking.hpp:11-17. Accepted and validated for API
 * compatibility; GPU tiling is internal. */
typedef struct cgb_blocking_params {
    int64_t mc, nc, kc, mr, nr;
} cgb_blocking_params;

typedef enum cgb_status {
    CGB_OK = 0,
    CGB_INVALID_GEOMETRY = 1,   /* InvalidGeometry   types.hpp:15 */
    CGB_DIMENSION_MISMATCH = 2, /* DimensionMismatch types.hpp:19 */
    CGB_ALLOCATION_FAILURE = 3, /* AllocationFailure types.hpp:23 */
    CGB_INVALID_ARGUMENT = 4,   /* std::invalid_argument blocking.hpp:24-28 */
    CGB_CUDA_ERROR = 5,         /* device/runtime failure (no reference equivalent) */
    CGB_UNSUPPORTED = 6         /* e.g. f64 requested on the device path */
} cgb_status;

/* Operator selection: the reference's Algo::Im2col / Algo::ConvGemm / Algo::Direct
 * (bench.hpp:13-19; conv.hpp:24-91). */
typedef enum cgb_algo {
    CGB_ALGO_EXPLICIT = 0, /* im2col kernel writes B-hat to HBM, then the GEMM kernel */
    CGB_ALGO_FUSED = 1,    /* implicit GEMM: B-hat tiles gathered straight into shared memory */
    CGB_ALGO_DIRECT = 2    /* conv_direct: the seven-loop convolution, bit-identical to the
                              reference's (fp32 product then add, its loop order); precision
                              is ignored. The checker, not a fast path. */
} cgb_algo;

/* Arithmetic on the tensor cores (or CUDA cores). */
typedef enum cgb_precision {
    CGB_PREC_AUTO = 0,   /* fp32-accurate: 3xTF32, or FFMA for degenerate low-K layers */
    CGB_PREC_3XTF32 = 1, /* split hi/lo TF32, 3 MMAs per k-step; tolerance 1e-5 (per-output normalised) */
    CGB_PREC_TF32 = 2,   /* plain TF32 tensor cores; tolerance 5e-3 (per-output normalised) */
    CGB_PREC_FFMA = 3    /* fp32 FFMA on CUDA cores; tolerance 1e-5 */
} cgb_precision;

/* ---- geometry (host only, conv_params.hpp / im2col.hpp) ---- */
cgb_status cgb_output_dims(const cgb_conv_params* cp, int64_t* h_o, int64_t* w_o);
cgb_status cgb_gemm_dims(const cgb_conv_params* cp, int64_t* m, int64_t* n, int64_t* k);
int64_t cgb_im2col_workspace_bytes(const cgb_conv_params* cp); /* k*n*4, im2col.hpp:36-39 (-1 on bad geometry) */
cgb_status cgb_validate_blocking(const cgb_blocking_params* bp);

/* Device workspace (bytes) the given call needs. The fused path needs none in
 * TF32 mode; 3xTF32 needs the filter hi/lo split (2*|F|); the explicit path
 * additionally holds B-hat (k x n). Pass workspace=NULL to cgb_conv* to let the
 * library use its own tracked, cached device allocation. */
int64_t cgb_conv_workspace_bytes(int algo, int precision, const cgb_conv_params* cp);
/* The same for cgb_gemm (C m x n = A m x k * B k x n, aligned B): the filter hi/lo split
 * of A for 3xTF32 when A is small; none in TF32 mode, and none for large A (> 8 MB: fc
 * weights), whose lo tile is split inside the kernel. -1 on bad dimensions. */
int64_t cgb_gemm_workspace_bytes(int precision, int64_t m, int64_t n, int64_t k);

/* ---- device-pointer entry points (asynchronous on `stream`) ---- */
cgb_status cgb_conv(int algo, int precision, const float* F, const float* I,
                    const cgb_conv_params* cp, float* O,
                    void* workspace, size_t workspace_bytes, void* stream);

/* Reference-named conveniences: bp may be NULL (= BlockingParams{}), threads is
 * accepted and ignored (the reference's team size, threads.hpp:29-42). */
cgb_status cgb_conv_gemm(const float* F, const float* I, const cgb_conv_params* cp,
                         const cgb_blocking_params* bp, int threads, float* O,
                         int precision, void* stream);
cgb_status cgb_conv_im2col_gemm(const float* F, const float* I, const cgb_conv_params* cp,
                                const cgb_blocking_params* bp, int threads, float* O,
                                int precision, void* stream);

/* Explicit lowered matrix B (k x n, column-major, leading dimension ldb >= k),
 * bit-identical to im2col<float>. Rows k..ldb-1 of each column are zero-filled. */
cgb_status cgb_im2col(const float* I, const cgb_conv_params* cp, float* B, int64_t ldb, void* stream);

/* C (m x n) = A (m x k) * B (k x n), column-major, O overwritten (the reference
 * zero-fills C before gemm, bench.cpp:149-151). Dense A and C (lda == ldc == m),
 * ldb >= k. Runs the explicit path's TMA-fed tensor-core GEMM (K2; FFMA for
 * CGB_PREC_FFMA) with B as the lowered matrix; few-column shapes (fc layers) are split
 * over K so every SM streams its share of A, partial tiles summed in a fixed order.
 * In the fp32-accurate mode weights larger than 8 MB are split into hi/lo in shared
 * memory (no workspace, no per-call pass over A). precision as for cgb_conv. */
cgb_status cgb_gemm(int precision, const float* A, int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                    int64_t m, int64_t n, int64_t k, void* workspace, size_t workspace_bytes, void* stream);

/* ---- host-pointer entry points: synchronous, reference semantics ----
 * Copies F and I host->device, runs cgb_conv, copies O device->host, syncs.
 * Host buffers may be pageable or pinned. */
cgb_status cgb_conv_host(int algo, int precision, const float* F_host, const float* I_host,
                         const cgb_conv_params* cp, float* O_host, void* stream);
/* im2col<float> (im2col.hpp:77-120) on host buffers: B_host (k x n, leading dimension
 * ldb >= k) written bit-identically to the reference's lowered matrix. */
cgb_status cgb_im2col_host(const float* I_host, const cgb_conv_params* cp, float* B_host, int64_t ldb);
/* gemm (gemm.hpp:46-105) on host buffers: C (+)= A * B for column-major A (m x k, lda),
 * B (k x n, ldb), C (m x n, ldc). accumulate != 0 adds to C like the reference's gemm
 * (which callers precede with zero_matrix); 0 overwrites C. */
cgb_status cgb_gemm_host(int precision, const float* A_host, int64_t lda, const float* B_host, int64_t ldb,
                         float* C_host, int64_t ldc, int64_t m, int64_t n, int64_t k, int accumulate);

/* ---- float64: the reference's f64 instantiations (bindings.cpp:58-65) on the device ----
 * Bit-identical to the reference's conv_direct<double> / conv_gemm<double> /
 * conv_im2col_gemm<double> / im2col<double> / gemm<double>: the reference's
 * accumulation order (kc-blocked, kc from bp; bp may be NULL = BlockingParams{}) with
 * every product rounded before its add, on FP64 CUDA cores. A checker and a
 * compatibility path, not the performance path. cgb_conv_f64 takes device pointers (on
 * `stream`); the *_host_f64 calls take host pointers and are synchronous. */
cgb_status cgb_conv_f64(int algo, const double* F, const double* I, const cgb_conv_params* cp,
                        const cgb_blocking_params* bp, double* O, void* stream);
cgb_status cgb_conv_host_f64(int algo, const double* F_host, const double* I_host, const cgb_conv_params* cp,
                             const cgb_blocking_params* bp, double* O_host);
cgb_status cgb_im2col_host_f64(const double* I_host, const cgb_conv_params* cp, double* B_host, int64_t ldb);
cgb_status cgb_gemm_host_f64(const double* A_host, int64_t lda, const double* B_host, int64_t ldb, double* C_host,
                             int64_t ldc, int64_t m, int64_t n, int64_t k, const cgb_blocking_params* bp,
                             int accumulate);

/* ---- workspace accounting (ScratchTracker equivalent, scratch.hpp:14-28) ----
 * Every call that needs device workspace (and was given none) claims its size: the
 * claim is checked against the limit on every call (non-zero limit -> oversized claims
 * fail with CGB_ALLOCATION_FAILURE, scratch.cpp:15-19) and counted in current/peak
 * while the call runs on the host (current returns to 0 between calls). The library
 * caches one buffer per (device, stream); buffers used while a stream was being
 * captured into a CUDA graph are never freed implicitly. */
uint64_t cgb_scratch_current_bytes(void);
uint64_t cgb_scratch_peak_bytes(void);
void cgb_scratch_reset_peak(void);
void cgb_scratch_set_limit(uint64_t bytes);
/* Free every cached workspace buffer (graphs captured earlier must not be replayed). */
void cgb_scratch_release(void);
/* Bytes currently held by the per-(device, stream) workspace caches. */
uint64_t cgb_scratch_cached_bytes(void);

/* ---- dispatch policy (no reference equivalent: the reference's BlockingParams are
 * CPU cache blocking, validated and otherwise ignored here) ----
 * Keys: "sk" (stream-K: 0 never, 1 auto, 2 always, 3 auto also for 1x1 layers), "tail" (tail tiles: 0/1/2), "pair"
 * (CTA pairs: 0 never, 1 by policy, 2 also for the low-channel w-im2col layers), "cfg" (force a kernel candidate, -1 auto), "mt", "bn" (force
 * tile sizes, 0 auto), "tma_a", "tma_deep" (1x1-layer variants), "pstore", "pdl",
 * "verbose", "smem_pad_kb", "tps", "splitk", "k2_flo" (explicit 3xTF32: filter lo tile split in
 * the kernel: -1 never, 0 by size, 1 always), "b_res" (filters resident in the ring when they fit), "urot" (rotate the window unit ->
 * staging warp assignment per chunk), "sk_pen_pct" (M-tile cost model: cost factor in percent of a stream-K split that reaches every tile,
 * filter tiles <= 128; default 130), "strip_h" (h-strips of that many output rows for wide stride-1 images:
 * 0 by rule, -1 off), "waste_pct" (cap on the shifted window's padded-plane rows per
 * output row in percent; 0 = none, the default), "host_chunk_kb", "host_no_bounce", "host_copy_threads",
 * "debug" (profiling builds only). Every setting gives a correct result; unknown keys
 * return CGB_INVALID_ARGUMENT. The library reads no environment variables. */
cgb_status cgb_set_tuning(const char* key, int64_t value);
cgb_status cgb_get_tuning(const char* key, int64_t* value);

/* ---- diagnostics ---- */
const char* cgb_last_error(void);
const char* cgb_version(void);
/* Number of device kernels this library launched since load (all entry points). */
uint64_t cgb_kernel_launch_count(void);
/* Kernel path the last cgb_conv chose on this thread: 0 none, 1 tcgen05 implicit,
 * 2 tcgen05 explicit, 3 ffma implicit, 4 ffma explicit. */
int cgb_last_path(void);
/* Profiling hook (profiling builds, -DCGB_PROFILING; returns -1 otherwise): per-CTA
 * MMA-issuer cycle counters of the last shifted-window launch made with debug & 64 set
 * (16 uint64 per CTA: total, wait accumulator, wait A window, wait filter tile, tiles,
 * epilogue wait/busy, timestamps). Returns 0 on success. */
int cgb_debug_sw_stats(unsigned long long* host, int n_cta);

#ifdef __cplusplus
}
#endif
#endif /* CONVGEMM_B200_H */
