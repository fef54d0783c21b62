// convgemm/conv.hpp -- drop-in for proj/include/convgemm/conv.hpp:9-119: the three
// convolution operators over host tensors, synchronous, O fully overwritten, on the B200:
//   conv_direct       the seven-loop reference, bit-identical to the reference's (float
//                     and double) -- the checker;
//   conv_im2col_gemm  explicit path: B-hat materialised in HBM, then the GEMM kernel;
//   conv_gemm         fused path: B-hat tiles staged straight into shared memory.
// float: tensor cores at convgemm::precision() (default fp32-accurate 3xTF32); double:
// the reference's f64 arithmetic bit for bit on FP64 cores.
#pragma once

#include <type_traits>

#include "convgemm/gemm.hpp"
#include "convgemm/im2col.hpp"
#include "convgemm/tensor.hpp"

namespace convgemm {

template <typename T>
void require_filter_shape(Tensor4View<const T> F, const ConvParams& cp) {
    if (F.d0 != cp.k_n || F.d1 != cp.k_h || F.d2 != cp.k_w || F.d3 != cp.c_i)
        throw InvalidGeometry("filter tensor extents disagree with ConvParams");
}

template <typename T>
void require_output_shape(Tensor4View<T> O, const ConvParams& cp, const OutputDims& od) {
    if (O.d0 != cp.k_n || O.d1 != od.h_o || O.d2 != od.w_o || O.d3 != cp.b)
        throw InvalidGeometry("output tensor extents disagree with ConvParams");
}

namespace detail {
template <typename T>
void run_conv(int algo, Tensor4View<const T> F, Tensor4View<const T> I, const ConvParams& cp,
              const BlockingParams& bp, Tensor4View<T> O) {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "convgemm: float or double");
    require_input_shape(I, cp);
    require_filter_shape(F, cp);
    require_output_shape(O, cp, output_dims(cp));
    validate(bp);
    const cgb_conv_params c = c_params(cp);
    if constexpr (std::is_same_v<T, float>) {
        check(cgb_conv_host(algo, static_cast<int>(precision()), F.data, I.data, &c, O.data, nullptr));
    } else {
        const cgb_blocking_params b = c_blocking(bp);
        check(cgb_conv_host_f64(algo, F.data, I.data, &c, &b, O.data));
    }
}
}  // namespace detail

template <typename T>
void conv_direct(Tensor4View<const T> F, Tensor4View<const T> I, const ConvParams& cp, Tensor4View<T> O) {
    detail::run_conv<T>(CGB_ALGO_DIRECT, F, I, cp, BlockingParams{}, O);
}

template <typename T>
void conv_im2col_gemm(Tensor4View<const T> F, Tensor4View<const T> I, const ConvParams& cp, const BlockingParams& bp,
                      int threads, Tensor4View<T> O) {
    (void)threads;
    detail::run_conv<T>(CGB_ALGO_EXPLICIT, F, I, cp, bp, O);
}

template <typename T>
void conv_gemm(Tensor4View<const T> F, Tensor4View<const T> I, const ConvParams& cp, const BlockingParams& bp,
               int threads, Tensor4View<T> O) {
    (void)threads;
    detail::run_conv<T>(CGB_ALGO_FUSED, F, I, cp, bp, O);
}

// owning forms (conv.hpp:93-119)
template <typename T>
Tensor4<T> conv_direct(const Tensor4<T>& F, const Tensor4<T>& I, const ConvParams& cp) {
    const OutputDims od = output_dims(cp);
    Tensor4<T> O(cp.k_n, od.h_o, od.w_o, cp.b);
    conv_direct<T>(F.view(), I.view(), cp, O.view());
    return O;
}

template <typename T>
Tensor4<T> conv_im2col_gemm(const Tensor4<T>& F, const Tensor4<T>& I, const ConvParams& cp,
                            const BlockingParams& bp = {}, int threads = 1) {
    const OutputDims od = output_dims(cp);
    Tensor4<T> O(cp.k_n, od.h_o, od.w_o, cp.b);
    conv_im2col_gemm<T>(F.view(), I.view(), cp, bp, threads, O.view());
    return O;
}

template <typename T>
Tensor4<T> conv_gemm(const Tensor4<T>& F, const Tensor4<T>& I, const ConvParams& cp, const BlockingParams& bp = {},
                     int threads = 1) {
    const OutputDims od = output_dims(cp);
    Tensor4<T> O(cp.k_n, od.h_o, od.w_o, cp.b);
    conv_gemm<T>(F.view(), I.view(), cp, bp, threads, O.view());
    return O;
}

}  // namespace convgemm
