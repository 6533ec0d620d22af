// attn_tc.cu — tcgen05/TMEM/TMA block-sparse attention forward (placeholder
// until the kernel lands; the dispatcher falls back to the mma.sync path).
#include <cuda_runtime.h>

#include "internal.h"

namespace blade {

size_t attn_tc_workspace(const AttnProblem&) { return 256; }

cudaError_t launch_attn_tc(const AttnProblem&, const void*, const void*, const void*,
                           const int32_t*, const int32_t*, void*, float*, char*, size_t,
                           cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace blade
