// convgemm/types.hpp -- drop-in for the reference's proj/include/convgemm/types.hpp:
// the index type and the exception vocabulary of the convgemm API, backed by the B200
// operator (libconvgemm_b200.so, include/convgemm_b200.h).
//
// This header tree (include/convgemm/*.hpp) keeps the reference's header names,
// namespace, type names, template signatures and call semantics (synchronous calls on
// host memory, O fully overwritten, the same exceptions), so reference callers --
// proj/src/bench.cpp and model.cpp are compiled unchanged against it in
// tests/test_cpp_dropin.py -- switch to the GPU by changing their include path and
// linking -lconvgemm_b200. float runs the tensor-core operator (fp32-accurate 3xTF32 by
// default, see convgemm::set_precision); double runs the reference's own f64 arithmetic
// bit for bit on the device's FP64 cores.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

#include "convgemm_b200.h"

namespace convgemm {

using index_t = std::int64_t;  // signed: padded coordinates go negative

inline constexpr index_t ceil_div(index_t a, index_t b) { return (a + b - 1) / b; }

struct InvalidGeometry : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct DimensionMismatch : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct AllocationFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ParseError : std::runtime_error {
    ParseError(int line_no, const std::string& what)
        : std::runtime_error("line " + std::to_string(line_no) + ": " + what), line(line_no) {}
    int line;
};
struct UnknownLayerKind : ParseError {
    UnknownLayerKind(int line_no, const std::string& kind) : ParseError(line_no, "unknown layer kind '" + kind + "'") {}
};
// B200 additions: a device/runtime failure, and a request the device path does not serve.
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct Unsupported : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

namespace detail {
// C-ABI status -> the reference's exception types (status codes: convgemm_b200.h)
inline void check(cgb_status st) {
    if (st == CGB_OK) return;
    const std::string msg = cgb_last_error();
    switch (st) {
        case CGB_INVALID_GEOMETRY: throw InvalidGeometry(msg);
        case CGB_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
        case CGB_ALLOCATION_FAILURE: throw AllocationFailure(msg);
        case CGB_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case CGB_UNSUPPORTED: throw Unsupported(msg);
        default: throw DeviceError(msg);
    }
}
}  // namespace detail

// Arithmetic of the float operators (the reference's float path is IEEE fp32; the
// default keeps fp32 accuracy on the tensor cores). Process-wide; not thread-local.
enum class Precision : int { Auto = CGB_PREC_AUTO, TF32x3 = CGB_PREC_3XTF32, TF32 = CGB_PREC_TF32, FFMA = CGB_PREC_FFMA };
namespace detail {
inline Precision& precision_ref() {
    static Precision p = Precision::Auto;
    return p;
}
}  // namespace detail
inline void set_precision(Precision p) { detail::precision_ref() = p; }
inline Precision precision() { return detail::precision_ref(); }

}  // namespace convgemm
