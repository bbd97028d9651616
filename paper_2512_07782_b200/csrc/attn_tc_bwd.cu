// attn_tc_bwd.cu -- tcgen05 backward (not yet enabled; SIMT path serves BF16).
#include "attn_common.cuh"

namespace gfwa {
bool tc_bwd_supported(const AttnParams&, gfwa_dtype_t) { return false; }
size_t tc_bwd_workspace(const AttnParams&) { return 0; }
gfwa_status_t tc_bwd(const AttnParams&, cudaStream_t, void*) { return GFWA_ERR_UNSUPPORTED; }
}  // namespace gfwa
