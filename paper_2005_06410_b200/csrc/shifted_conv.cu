// shifted_conv.cu -- V2 "shifted window" tcgen05 kernel (stride-phase staging, taps as
// shared-memory descriptor row offsets). Not yet enabled: shifted_supported() gates it.
#include "internal.h"

namespace cgb {

bool shifted_supported(const ConvGeom&) { return false; }

cudaError_t launch_tc_conv_shifted(const float*, const float*, int64_t, const float*, float*, const ConvGeom&, bool,
                                   cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace cgb
