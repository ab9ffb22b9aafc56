// window_tiled.cu — tiled window/dilated kernel (placeholder until implemented).
#include "common.cuh"

namespace ga {

bool window_tiled_supported(const AttnParams &, ga_dtype) { return false; }

ga_status launch_window_tiled(const AttnParams &, ga_dtype, cudaStream_t)
{
    set_error("tiled window kernel not built");
    return GA_ERR_UNSUPPORTED;
}

} // namespace ga
