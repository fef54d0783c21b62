// convgemm_b200.hpp -- C++ drop-in shim: the reference's convgemm API names for float,
// forwarding to the C-ABI in convgemm_b200.h (device path) with the reference's
// synchronous, host-memory call semantics.
//
// A reference caller (proj/src/bench.cpp:166-196, proj/tests/*.cpp) that does
//     #include "convgemm/conv.hpp"
//     convgemm::conv_gemm<float>(F, I, cp, bp, threads, O);
// switches to the B200 operator by including this header instead and using
// namespace convgemm_b200 (or `namespace convgemm = convgemm_b200;`). Views,
// ConvParams, BlockingParams, the owning Tensor4 and the exception types have the
// reference's names, fields and semantics (tensor.hpp:12-123, conv_params.hpp:8-43,
// blocking.hpp:11-29, types.hpp:15-41); O is fully overwritten (conv.hpp:71,89).
//
// Header-only; link with paper_2005_06410_b200/libconvgemm_b200.so.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "convgemm_b200.h"

namespace convgemm_b200 {

using index_t = std::int64_t;

struct InvalidGeometry : std::runtime_error { using std::runtime_error::runtime_error; };
struct DimensionMismatch : std::runtime_error { using std::runtime_error::runtime_error; };
struct AllocationFailure : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

// Precision of the B200 operator (the reference is fp32 throughout; Auto keeps fp32 accuracy).
enum class Precision : int { Auto = CGB_PREC_AUTO, TF32x3 = CGB_PREC_3XTF32, TF32 = CGB_PREC_TF32, FFMA = CGB_PREC_FFMA };

struct ConvParams {  // conv_params.hpp:8-16
  index_t k_n = 1, k_h = 1, k_w = 1, c_i = 1, h_i = 1, w_i = 1, b = 1, s = 1, p = 0;
  cgb_conv_params c() const { return {k_n, k_h, k_w, c_i, h_i, w_i, b, s, p}; }
};
struct OutputDims { index_t h_o = 0, w_o = 0; };
struct GemmDims { index_t m = 0, n = 0, k = 0; };
struct BlockingParams {  // blocking.hpp:11-17
  index_t mc = 120, nc = 3072, kc = 640, mr = 8, nr = 12;
  cgb_blocking_params c() const { return {mc, nc, kc, mr, nr}; }
};

inline void throw_on(cgb_status st) {
  if (st == CGB_OK) return;
  const std::string msg = cgb_last_error();
  switch (st) {
    case CGB_INVALID_GEOMETRY: throw InvalidGeometry(msg);
    case CGB_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case CGB_ALLOCATION_FAILURE: throw AllocationFailure(msg);
    case CGB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw DeviceError(msg);
  }
}

inline OutputDims output_dims(const ConvParams& cp) {  // conv_params.hpp:27-36
  const cgb_conv_params c = cp.c();
  OutputDims od;
  throw_on(cgb_output_dims(&c, &od.h_o, &od.w_o));
  return od;
}

inline GemmDims gemm_dims(const ConvParams& cp) {  // conv_params.hpp:40-43
  const cgb_conv_params c = cp.c();
  GemmDims g;
  throw_on(cgb_gemm_dims(&c, &g.m, &g.n, &g.k));
  return g;
}

inline index_t im2col_workspace_bytes(const ConvParams& cp) {  // im2col.hpp:36-39
  output_dims(cp);
  const cgb_conv_params c = cp.c();
  return cgb_im2col_workspace_bytes(&c);
}

inline void validate(const BlockingParams& bp) {  // blocking.hpp:22-29
  const cgb_blocking_params c = bp.c();
  throw_on(cgb_validate_blocking(&c));
}

// Leftmost-fastest rank-4 view, tensor.hpp:30-50.
template <typename T>
struct Tensor4View {
  T* data = nullptr;
  index_t d0 = 0, d1 = 0, d2 = 0, d3 = 0;
  index_t size() const { return d0 * d1 * d2 * d3; }
  index_t offset(index_t i0, index_t i1, index_t i2, index_t i3) const { return i0 + d0 * (i1 + d1 * (i2 + d2 * i3)); }
  T& operator()(index_t i0, index_t i1, index_t i2, index_t i3) const { return data[offset(i0, i1, i2, i3)]; }
  operator Tensor4View<const T>() const { return {data, d0, d1, d2, d3}; }
};

// Owning zero-initialised rank-4 tensor, tensor.hpp:54-88.
template <typename T>
class Tensor4 {
 public:
  Tensor4(index_t d0, index_t d1, index_t d2, index_t d3) : d0_(d0), d1_(d1), d2_(d2), d3_(d3) {
    if (d0 < 1 || d1 < 1 || d2 < 1 || d3 < 1) throw InvalidGeometry("tensor extents must be positive");
    data_.assign(static_cast<std::size_t>(d0 * d1 * d2 * d3), T(0));
  }
  index_t d0() const { return d0_; }
  index_t d1() const { return d1_; }
  index_t d2() const { return d2_; }
  index_t d3() const { return d3_; }
  index_t size() const { return static_cast<index_t>(data_.size()); }
  T* data() { return data_.data(); }
  const T* data() const { return data_.data(); }
  T& operator()(index_t i0, index_t i1, index_t i2, index_t i3) { return data_[view().offset(i0, i1, i2, i3)]; }
  const T& operator()(index_t i0, index_t i1, index_t i2, index_t i3) const {
    return data_[view().offset(i0, i1, i2, i3)];
  }
  Tensor4View<T> view() { return {data_.data(), d0_, d1_, d2_, d3_}; }
  Tensor4View<const T> view() const { return {data_.data(), d0_, d1_, d2_, d3_}; }

 private:
  index_t d0_, d1_, d2_, d3_;
  std::vector<T> data_;
};

namespace detail {
inline void require_shapes(Tensor4View<const float> F, Tensor4View<const float> I, Tensor4View<float> O,
                           const ConvParams& cp) {  // conv.hpp:9-19, im2col.hpp:46-50
  const OutputDims od = output_dims(cp);
  if (I.d0 != cp.h_i || I.d1 != cp.w_i || I.d2 != cp.c_i || I.d3 != cp.b)
    throw InvalidGeometry("input tensor extents disagree with ConvParams");
  if (F.d0 != cp.k_n || F.d1 != cp.k_h || F.d2 != cp.k_w || F.d3 != cp.c_i)
    throw InvalidGeometry("filter tensor extents disagree with ConvParams");
  if (O.d0 != cp.k_n || O.d1 != od.h_o || O.d2 != od.w_o || O.d3 != cp.b)
    throw InvalidGeometry("output tensor extents disagree with ConvParams");
}

inline void run(int algo, Tensor4View<const float> F, Tensor4View<const float> I, const ConvParams& cp,
                const BlockingParams& bp, Tensor4View<float> O, Precision prec) {
  validate(bp);
  require_shapes(F, I, O, cp);
  const cgb_conv_params c = cp.c();
  throw_on(cgb_conv_host(algo, static_cast<int>(prec), F.data, I.data, &c, O.data, nullptr));
}
}  // namespace detail

// conv.hpp:60-74 -- explicit im2col + GEMM (B-hat materialised in HBM).
inline void conv_im2col_gemm(Tensor4View<const float> F, Tensor4View<const float> I, const ConvParams& cp,
                             const BlockingParams& bp, int /*threads*/, Tensor4View<float> O,
                             Precision prec = Precision::Auto) {
  detail::run(CGB_ALGO_EXPLICIT, F, I, cp, bp, O, prec);
}

// conv.hpp:78-91 -- fused ConvGemm (B-hat tiles gathered straight into shared memory).
inline void conv_gemm(Tensor4View<const float> F, Tensor4View<const float> I, const ConvParams& cp,
                      const BlockingParams& bp, int /*threads*/, Tensor4View<float> O,
                      Precision prec = Precision::Auto) {
  detail::run(CGB_ALGO_FUSED, F, I, cp, bp, O, prec);
}

// Owning overloads, conv.hpp:101-119.
inline Tensor4<float> conv_im2col_gemm(const Tensor4<float>& F, const Tensor4<float>& I, const ConvParams& cp,
                                       const BlockingParams& bp = {}, int threads = 1,
                                       Precision prec = Precision::Auto) {
  const OutputDims od = output_dims(cp);
  Tensor4<float> O(cp.k_n, od.h_o, od.w_o, cp.b);
  conv_im2col_gemm(F.view(), I.view(), cp, bp, threads, O.view(), prec);
  return O;
}

inline Tensor4<float> conv_gemm(const Tensor4<float>& F, const Tensor4<float>& I, const ConvParams& cp,
                                const BlockingParams& bp = {}, int threads = 1, Precision prec = Precision::Auto) {
  const OutputDims od = output_dims(cp);
  Tensor4<float> O(cp.k_n, od.h_o, od.w_o, cp.b);
  conv_gemm(F.view(), I.view(), cp, bp, threads, O.view(), prec);
  return O;
}

}  // namespace convgemm_b200
