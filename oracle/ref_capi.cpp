// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A C-ABI shim over the UNMODIFIED reference library so that Python tests and
// the bench's CPU-baseline / reference arm can call the reference's own conv
// operator. The reference is header-only (proj/include/convgemm/*.hpp) plus
// proj/src/scratch.cpp; both are compiled from where they lie under
// /root/reference by oracle/Makefile into oracle/_ref/ (git-ignored).
// Nothing here re-implements reference arithmetic: every entry forwards to a
// reference template:
//   conv_direct        proj/include/convgemm/conv.hpp:24-55
//   conv_im2col_gemm   proj/include/convgemm/conv.hpp:60-74
//   conv_gemm          proj/include/convgemm/conv.hpp:78-91
//   im2col             proj/include/convgemm/im2col.hpp:77-120
//   gemm               proj/include/convgemm/gemm.hpp:100-105
//   output_dims        proj/include/convgemm/conv_params.hpp:27-36
//   random generators  proj/tests/oracles.hpp:48-91 (mt19937_64 streams)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <random>
#include <stdexcept>
#include <string>

#include "convgemm/conv.hpp"
#include "convgemm/scratch.hpp"
#include "oracles.hpp"

using namespace convgemm;

namespace {
thread_local std::string g_last_error;

ConvParams to_cp(const int64_t* a) {
    ConvParams cp;
    cp.k_n = a[0]; cp.k_h = a[1]; cp.k_w = a[2]; cp.c_i = a[3];
    cp.h_i = a[4]; cp.w_i = a[5]; cp.b = a[6]; cp.s = a[7]; cp.p = a[8];
    return cp;
}

BlockingParams to_bp(const int64_t* a) {
    BlockingParams bp;
    if (a) { bp.mc = a[0]; bp.nc = a[1]; bp.kc = a[2]; bp.mr = a[3]; bp.nr = a[4]; }
    return bp;
}

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const InvalidGeometry& e) {
        g_last_error = e.what(); return 1;
    } catch (const DimensionMismatch& e) {
        g_last_error = e.what(); return 2;
    } catch (const AllocationFailure& e) {
        g_last_error = e.what(); return 3;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what(); return 4;
    } catch (const std::exception& e) {
        g_last_error = e.what(); return 9;
    }
}

template <typename T>
void run(int kind, const void* F, const void* I, const int64_t* cpa, const int64_t* bpa,
         int threads, void* O) {
    const ConvParams cp = to_cp(cpa);
    const BlockingParams bp = to_bp(bpa);
    const OutputDims od = output_dims(cp);
    Tensor4View<const T> Fv{static_cast<const T*>(F), cp.k_n, cp.k_h, cp.k_w, cp.c_i};
    Tensor4View<const T> Iv{static_cast<const T*>(I), cp.h_i, cp.w_i, cp.c_i, cp.b};
    Tensor4View<T> Ov{static_cast<T*>(O), cp.k_n, od.h_o, od.w_o, cp.b};
    switch (kind) {
        case 0: conv_direct<T>(Fv, Iv, cp, Ov); break;
        case 1: conv_im2col_gemm<T>(Fv, Iv, cp, bp, threads, Ov); break;
        case 2: conv_gemm<T>(Fv, Iv, cp, bp, threads, Ov); break;
        default: throw std::invalid_argument("unknown conv kind");
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// kind: 0 = conv_direct, 1 = conv_im2col_gemm, 2 = conv_gemm; dtype: 0 f32, 1 f64.
int ref_conv(int kind, int dtype, const void* F, const void* I, const int64_t* cp,
             const int64_t* bp, int threads, void* O) {
    return guarded([&] {
        if (dtype == 0) run<float>(kind, F, I, cp, bp, threads, O);
        else run<double>(kind, F, I, cp, bp, threads, O);
    });
}

int ref_output_dims(const int64_t* cp, int64_t* h_o, int64_t* w_o) {
    return guarded([&] {
        const OutputDims od = output_dims(to_cp(cp));
        *h_o = od.h_o; *w_o = od.w_o;
    });
}

int ref_gemm_dims(const int64_t* cp, int64_t* m, int64_t* n, int64_t* k) {
    return guarded([&] {
        const GemmDims g = gemm_dims(to_cp(cp));
        *m = g.m; *n = g.n; *k = g.k;
    });
}

int64_t ref_im2col_workspace_bytes(const int64_t* cp) { return im2col_workspace_bytes(to_cp(cp)); }
int64_t ref_convgemm_scratch_bytes(const int64_t* bp) { return convgemm_scratch_bytes(to_bp(bp)); }

// Explicit lowered matrix B (k x n, ld = k), exactly as im2col<float> returns it.
int ref_im2col_f32(const float* I, const int64_t* cpa, int threads, float* B) {
    return guarded([&] {
        const ConvParams cp = to_cp(cpa);
        Tensor4View<const float> Iv{I, cp.h_i, cp.w_i, cp.c_i, cp.b};
        const Im2colMatrix<float> m = im2col<float>(Iv, cp, threads);
        std::copy_n(m.view().data, m.rows() * m.cols(), B);
    });
}

int ref_im2col_f64(const double* I, const int64_t* cpa, int threads, double* B) {
    return guarded([&] {
        const ConvParams cp = to_cp(cpa);
        Tensor4View<const double> Iv{I, cp.h_i, cp.w_i, cp.c_i, cp.b};
        const Im2colMatrix<double> m = im2col<double>(Iv, cp, threads);
        std::copy_n(m.view().data, m.rows() * m.cols(), B);
    });
}

int ref_gemm_f64(const double* A, const double* B, double* C, int64_t m, int64_t n, int64_t k,
                 const int64_t* bp, int threads) {
    return guarded([&] {
        MatrixView<double> Cv{C, m, n, m};
        zero_matrix(Cv);
        gemm<double>(MatrixView<const double>{A, m, k, m}, MatrixView<const double>{B, k, n, k}, Cv,
                     to_bp(bp), threads);
    });
}

// Column-major C = A*B (m x k times k x n), reference blocked gemm.
int ref_gemm_f32(const float* A, const float* B, float* C, int64_t m, int64_t n, int64_t k,
                 const int64_t* bp, int threads) {
    return guarded([&] {
        MatrixView<float> Cv{C, m, n, m};
        zero_matrix(Cv);
        gemm<float>(MatrixView<const float>{A, m, k, m}, MatrixView<const float>{B, k, n, k}, Cv,
                    to_bp(bp), threads);
    });
}

// Pack-level equality hook (acceptance.cpp:89-135): fused pack vs pack over im2col.
// Returns number of mismatching macro-blocks, straddles through *straddles.
int64_t ref_pack_check(const float* I, const int64_t* cpa, const int64_t* bpa, int64_t* straddles) {
    const ConvParams cp = to_cp(cpa);
    const BlockingParams bp = to_bp(bpa);
    const OutputDims od = output_dims(cp);
    const GemmDims g = gemm_dims(cp);
    Tensor4View<const float> Iv{I, cp.h_i, cp.w_i, cp.c_i, cp.b};
    const auto lowered = im2col<float>(Iv, cp);
    MatrixSource<float> explicit_src(lowered.view());
    Im2colSource<float> fused_src(Iv, cp);
    PackedPanel<float> expect(bp.kc * bp.nc, bp.nr);
    PackedPanel<float> got(bp.kc * bp.nc, bp.nr);
    int64_t bad = 0;
    *straddles = 0;
    for (index_t j_c = 0; j_c < g.n; j_c += bp.nc) {
        const index_t nc_eff = std::min(bp.nc, g.n - j_c);
        if (j_c / (od.h_o * od.w_o) != (j_c + nc_eff - 1) / (od.h_o * od.w_o)) ++*straddles;
        for (index_t p_c = 0; p_c < g.k; p_c += bp.kc) {
            const index_t kc_eff = std::min(bp.kc, g.k - p_c);
            const index_t used = ceil_div(nc_eff, bp.nr) * bp.nr * kc_eff;
            std::fill_n(expect.data.data(), used, -3.0f);
            std::fill_n(got.data.data(), used, 3.0f);
            pack_b<float>(explicit_src, p_c, j_c, kc_eff, nc_eff, bp, expect);
            pack_b_im2col<float>(fused_src, p_c, j_c, kc_eff, nc_eff, bp, got);
            if (std::memcmp(got.data.data(), expect.data.data(),
                            static_cast<std::size_t>(used) * sizeof(float)) != 0)
                ++bad;
        }
    }
    return bad;
}

uint64_t ref_scratch_peak_bytes() { return ScratchTracker::peak_bytes(); }
void ref_scratch_reset_peak() { ScratchTracker::reset_peak(); }
void ref_scratch_set_limit(uint64_t bytes) { ScratchTracker::set_limit(bytes); }

// ---- the reference tests' seeded generators (tests/oracles.hpp) ----
void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* h) { delete static_cast<std::mt19937_64*>(h); }
void ref_rng_fill_uniform_f32(void* h, float* p, int64_t n) {
    testutil::fill_uniform(p, n, *static_cast<std::mt19937_64*>(h));
}
void ref_rng_fill_uniform_f64(void* h, double* p, int64_t n) {
    testutil::fill_uniform(p, n, *static_cast<std::mt19937_64*>(h));
}
void ref_rng_random_conv_params(void* h, int64_t cap, int64_t max_batch, int64_t* out) {
    const ConvParams cp = testutil::random_conv_params(*static_cast<std::mt19937_64*>(h), cap, max_batch);
    out[0] = cp.k_n; out[1] = cp.k_h; out[2] = cp.k_w; out[3] = cp.c_i;
    out[4] = cp.h_i; out[5] = cp.w_i; out[6] = cp.b; out[7] = cp.s; out[8] = cp.p;
}
int64_t ref_rng_rand_in(void* h, int64_t lo, int64_t hi) {
    return testutil::rand_in(*static_cast<std::mt19937_64*>(h), lo, hi);
}

}  // extern "C"
