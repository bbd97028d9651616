// attn_tc_fwd.cu -- tcgen05 forward (not yet enabled; SIMT path serves BF16).
#include "attn_common.cuh"

namespace gfwa {
bool tc_fwd_supported(const AttnParams&, gfwa_dtype_t) { return false; }
gfwa_status_t tc_fwd(const AttnParams&, cudaStream_t) { return GFWA_ERR_UNSUPPORTED; }
}  // namespace gfwa
