// tile.h -- fused window tile pass (filled in by tile_pass.cu).
#pragma once

#include "qj_internal.h"

namespace qj {

struct TileSpec {
    int dummy = 0;
};

template <typename R>
cudaError_t run_tile(const TileSpec& t, void* psi, int nl, cudaStream_t st, LaunchStats& ls);

}  // namespace qj
