// convgemm/blocking.hpp -- drop-in for proj/include/convgemm/blocking.hpp:11-29.
// The CPU cache/register blocking is accepted and validated with the reference's rules
// and messages (std::invalid_argument); the device tiling is internal. kc alone matters
// on the device: it is the accumulation block of the bit-exact float64 path.
#pragma once

#include <stdexcept>

#include "convgemm/types.hpp"

namespace convgemm {

struct BlockingParams {
    index_t mc = 120;
    index_t nc = 3072;
    index_t kc = 640;
    index_t mr = 8;
    index_t nr = 12;
};

inline constexpr index_t kMaxMicroTile = 4096;

namespace detail {
inline cgb_blocking_params c_blocking(const BlockingParams& bp) {
    return cgb_blocking_params{bp.mc, bp.nc, bp.kc, bp.mr, bp.nr};
}
}  // namespace detail

inline void validate(const BlockingParams& bp) {
    const cgb_blocking_params c = detail::c_blocking(bp);
    detail::check(cgb_validate_blocking(&c));
}

}  // namespace convgemm
