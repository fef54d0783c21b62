// convgemm_b200.hpp -- the C++ drop-in surface in one include: the reference's convgemm
// API (header tree include/convgemm/, same names and semantics as
// proj/include/convgemm/*.hpp) over the C-ABI in convgemm_b200.h. Reference callers
// include "convgemm/conv.hpp" etc. directly; this header also offers the namespace
// alias convgemm_b200.
#pragma once

#include "convgemm/bench.hpp"
#include "convgemm/conv.hpp"
#include "convgemm/gemm.hpp"
#include "convgemm/im2col.hpp"
#include "convgemm/model.hpp"
#include "convgemm/scratch.hpp"
#include "convgemm/threads.hpp"

namespace convgemm_b200 = convgemm;
