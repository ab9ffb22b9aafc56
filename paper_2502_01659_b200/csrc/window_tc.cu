// window_tc.cu — tcgen05 dense-tile window kernel (placeholder until implemented).
#include "common.cuh"

namespace ga {

bool window_tc_supported(const AttnParams &, ga_dtype) { return false; }

ga_status launch_window_tc(const AttnParams &, ga_dtype, cudaStream_t)
{
    set_error("tcgen05 window kernel not built");
    return GA_ERR_UNSUPPORTED;
}

} // namespace ga
