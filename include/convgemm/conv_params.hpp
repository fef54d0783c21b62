// convgemm/conv_params.hpp -- drop-in for proj/include/convgemm/conv_params.hpp:8-43.
// The geometry rules live in the library (cgb_output_dims / cgb_gemm_dims) so host and
// device agree on them; errors are the reference's InvalidGeometry.
#pragma once

#include "convgemm/types.hpp"

namespace convgemm {

struct ConvParams {
    index_t k_n = 1;           // filters
    index_t k_h = 1, k_w = 1;  // filter extents
    index_t c_i = 1;           // input channels
    index_t h_i = 1, w_i = 1;  // input extents
    index_t b = 1;             // batch
    index_t s = 1;             // stride
    index_t p = 0;             // symmetric zero padding
};

struct OutputDims {
    index_t h_o = 0, w_o = 0;
};

struct GemmDims {
    index_t m = 0, n = 0, k = 0;
};

namespace detail {
inline cgb_conv_params c_params(const ConvParams& cp) {
    return cgb_conv_params{cp.k_n, cp.k_h, cp.k_w, cp.c_i, cp.h_i, cp.w_i, cp.b, cp.s, cp.p};
}
}  // namespace detail

// h_o = floor((h_i - k_h + 2p) / s) + 1, likewise w_o; InvalidGeometry otherwise.
inline OutputDims output_dims(const ConvParams& cp) {
    const cgb_conv_params c = detail::c_params(cp);
    OutputDims od;
    detail::check(cgb_output_dims(&c, &od.h_o, &od.w_o));
    return od;
}

// m = k_n, n = h_o*w_o*b, k = k_h*k_w*c_i.
inline GemmDims gemm_dims(const ConvParams& cp) {
    const cgb_conv_params c = detail::c_params(cp);
    GemmDims g;
    detail::check(cgb_gemm_dims(&c, &g.m, &g.n, &g.k));
    return g;
}

}  // namespace convgemm
