// convgemm/gemm.hpp -- drop-in for proj/include/convgemm/gemm.hpp:11-105: zero_matrix
// and C += A * B over a PackingSource, on the device (float: tensor cores at
// convgemm::precision(); double: the reference's kc-blocked order bit for bit).
#pragma once

#include <algorithm>
#include <type_traits>
#include <vector>

#include "convgemm/conv_params.hpp"
#include "convgemm/im2col.hpp"
#include "convgemm/packing.hpp"

namespace convgemm {

// Work counters of the reference's blocked loops (gemm.hpp:11-23); the device fills flops.
struct GemmBlockStat {
    index_t kc_eff = 0, nc_eff = 0, b_elements_packed = 0, l3_flops = 0;
};
struct GemmStats {
    std::vector<GemmBlockStat> blocks;
    index_t a_elements_packed = 0;
    index_t flops = 0;
};

template <typename T>
void zero_matrix(MatrixView<T> C) {
    for (index_t j = 0; j < C.cols; ++j) std::fill_n(C.data + j * C.ld, C.rows, T(0));
}

namespace detail {
template <typename T>
void gemm_matrix(MatrixView<const T> A, MatrixView<const T> B, MatrixView<T> C, index_t m, index_t n, index_t k,
                 const BlockingParams& bp) {
    if constexpr (std::is_same_v<T, float>) {
        check(cgb_gemm_host(static_cast<int>(precision()), A.data, A.ld, B.data, B.ld, C.data, C.ld, m, n, k, 1));
    } else {
        const cgb_blocking_params b = c_blocking(bp);
        check(cgb_gemm_host_f64(A.data, A.ld, B.data, B.ld, C.data, C.ld, m, n, k, &b, 1));
    }
}
}  // namespace detail

// C += A * B (callers zero C first, as the reference's operators do).
template <typename T>
void gemm(MatrixView<const T> A, const PackingSource<T>& B, MatrixView<T> C, const GemmDims& dims,
          const BlockingParams& bp, int threads = 1, GemmStats* stats = nullptr) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "convgemm: float or double");
    (void)threads;
    validate(bp);
    if (A.rows != dims.m || A.cols != dims.k || C.rows != dims.m || C.cols != dims.n || B.rows() != dims.k ||
        B.cols() != dims.n)
        throw DimensionMismatch("gemm operand extents disagree with (m,n,k)");
    if (stats) stats->flops = 2 * dims.m * dims.n * dims.k;
    const detail::DeviceOperand<T> op = B.device_operand();
    if (op.kind == detail::DeviceOperand<T>::Matrix) {
        detail::gemm_matrix<T>(A, op.matrix, C, dims.m, dims.n, dims.k, bp);
        return;
    }
    std::vector<T> dense;  // the operand as a dense k x n matrix when the device cannot read it directly
    if (op.kind == detail::DeviceOperand<T>::Conv) {
        // the implicit convolution with A as its filters (A dense: ld == m is a k_n x K filter tensor)
        std::vector<T> Ad;
        const T* F = A.data;
        if (A.ld != A.rows) {
            Ad.resize(static_cast<std::size_t>(dims.m * dims.k));
            for (index_t j = 0; j < dims.k; ++j) std::copy_n(A.data + j * A.ld, dims.m, Ad.data() + j * dims.m);
            F = Ad.data();
        }
        std::vector<T> tmp(static_cast<std::size_t>(dims.m * dims.n));
        const cgb_conv_params c = detail::c_params(*op.conv);
        if constexpr (std::is_same_v<T, float>) {
            detail::check(cgb_conv_host(CGB_ALGO_FUSED, static_cast<int>(precision()), F, op.input, &c, tmp.data(), nullptr));
        } else {
            const cgb_blocking_params b = detail::c_blocking(bp);
            detail::check(cgb_conv_host_f64(CGB_ALGO_FUSED, F, op.input, &c, &b, tmp.data()));
        }
        for (index_t j = 0; j < dims.n; ++j)
            for (index_t i = 0; i < dims.m; ++i) C(i, j) += tmp[static_cast<std::size_t>(i + j * dims.m)];
        return;
    }
    dense.resize(static_cast<std::size_t>(dims.k * dims.n));
    for (index_t j = 0; j < dims.n; ++j)
        for (index_t i = 0; i < dims.k; ++i) dense[static_cast<std::size_t>(i + j * dims.k)] = B.at(i, j);
    detail::gemm_matrix<T>(A, MatrixView<const T>{dense.data(), dims.k, dims.n, dims.k}, C, dims.m, dims.n, dims.k, bp);
}

// Convenience form over a plain matrix (gemm.hpp:100-105).
template <typename T>
void gemm(MatrixView<const T> A, MatrixView<const T> B, MatrixView<T> C, const BlockingParams& bp = {}, int threads = 1) {
    gemm<T>(A, MatrixSource<T>(B), C, GemmDims{A.rows, B.cols, A.cols}, bp, threads);
}

}  // namespace convgemm
