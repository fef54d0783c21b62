// convgemm/im2col.hpp -- drop-in for proj/include/convgemm/im2col.hpp:9-167: the
// lowered-matrix coordinates, workspace formulas, the explicit transform (run by the
// device kernel, bit-identical: pure data movement) and the fused source.
#pragma once

#include <type_traits>
#include <vector>

#include "convgemm/conv_params.hpp"
#include "convgemm/packing.hpp"

namespace convgemm {

struct RowCoords {
    index_t i_c, i_kw, i_kh;
};
struct ColCoords {
    index_t i_b, i_w, i_h;
};

// r = i_kh + i_kw*k_h + i_c*k_h*k_w
inline RowCoords decompose_row(index_t r, const ConvParams& cp) {
    const index_t taps = cp.k_h * cp.k_w, t = r % taps;
    return {r / taps, t / cp.k_h, t % cp.k_h};
}
// c = i_h + i_w*h_o + i_b*h_o*w_o
inline ColCoords decompose_col(index_t c, const OutputDims& od) {
    const index_t plane = od.h_o * od.w_o, t = c % plane;
    return {c / plane, t / od.h_o, t % od.h_o};
}
inline ColCoords decompose_col(index_t c, const ConvParams& cp) { return decompose_col(c, output_dims(cp)); }

// k x n floats of the explicit path (im2col.hpp:36-39).
inline index_t im2col_workspace_bytes(const ConvParams& cp) {
    const cgb_conv_params c = detail::c_params(cp);
    output_dims(cp);  // InvalidGeometry first, as the reference
    return cgb_im2col_workspace_bytes(&c);
}

// The reference's fused-path packing buffers (im2col.hpp:41-44). The device fused path
// takes no workspace of its own in TF32 mode (the filter split in 3xTF32); this formula
// is kept for callers that report the reference's number.
inline index_t convgemm_scratch_bytes(const BlockingParams& bp) {
    return (bp.mc * bp.kc + bp.kc * bp.nc) * static_cast<index_t>(sizeof(float));
}

template <typename T>
void require_input_shape(Tensor4View<const T> I, const ConvParams& cp) {
    if (I.d0 != cp.h_i || I.d1 != cp.w_i || I.d2 != cp.c_i || I.d3 != cp.b)
        throw InvalidGeometry("input tensor extents disagree with ConvParams");
}

// Owning lowered matrix (k x n, ld = k) in host memory.
template <typename T>
class Im2colMatrix {
public:
    Im2colMatrix(index_t rows, index_t cols) : rows_(rows), cols_(cols), storage_(static_cast<std::size_t>(rows * cols)) {}
    index_t rows() const { return rows_; }
    index_t cols() const { return cols_; }
    MatrixView<T> view() { return {storage_.data(), rows_, cols_, rows_}; }
    MatrixView<const T> view() const { return {storage_.data(), rows_, cols_, rows_}; }

private:
    index_t rows_, cols_;
    std::vector<T> storage_;
};

// im2col<T> (im2col.hpp:77-120) on the device: I -> B-hat, identical to the reference's.
template <typename T>
Im2colMatrix<T> im2col(Tensor4View<const T> I, const ConvParams& cp, int threads = 1) {
    (void)threads;
    require_input_shape(I, cp);
    const GemmDims g = gemm_dims(cp);
    Im2colMatrix<T> out(g.k, g.n);
    const cgb_conv_params c = detail::c_params(cp);
    if constexpr (std::is_same_v<T, float>)
        detail::check(cgb_im2col_host(I.data, &c, out.view().data, g.k));
    else if constexpr (std::is_same_v<T, double>)
        detail::check(cgb_im2col_host_f64(I.data, &c, out.view().data, g.k));
    else
        static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "convgemm: float or double");
    return out;
}

// The lowered matrix served straight from I (im2col.hpp:132-167); on the device gemm()
// runs it as the fused implicit convolution.
template <typename T>
class Im2colSource final : public PackingSource<T> {
public:
    Im2colSource(Tensor4View<const T> I, const ConvParams& cp) : I_(I), cp_(cp), od_(output_dims(cp)) {
        require_input_shape(I, cp);
    }
    index_t rows() const override { return cp_.k_h * cp_.k_w * cp_.c_i; }
    index_t cols() const override { return od_.h_o * od_.w_o * cp_.b; }
    T at(index_t row, index_t col) const override {
        const RowCoords r = decompose_row(row, cp_);
        const ColCoords c = decompose_col(col, od_);
        const index_t h = c.i_h * cp_.s + r.i_kh - cp_.p, w = c.i_w * cp_.s + r.i_kw - cp_.p;
        if (h < 0 || h >= cp_.h_i || w < 0 || w >= cp_.w_i) return T(0);
        return I_(h, w, r.i_c, c.i_b);
    }
    detail::DeviceOperand<T> device_operand() const override {
        detail::DeviceOperand<T> d;
        d.kind = detail::DeviceOperand<T>::Conv;
        d.input = I_.data;
        d.conv = &cp_;
        return d;
    }

private:
    Tensor4View<const T> I_;
    ConvParams cp_;
    OutputDims od_;
};

}  // namespace convgemm
