// tile_pass.cu -- fused window tile pass (placeholder until the planner lands).
#include "tile.h"

namespace qj {
template <typename R>
cudaError_t run_tile(const TileSpec&, void*, int, cudaStream_t, LaunchStats&) {
    return cudaErrorNotSupported;
}
template cudaError_t run_tile<float>(const TileSpec&, void*, int, cudaStream_t, LaunchStats&);
template cudaError_t run_tile<double>(const TileSpec&, void*, int, cudaStream_t, LaunchStats&);
}  // namespace qj
