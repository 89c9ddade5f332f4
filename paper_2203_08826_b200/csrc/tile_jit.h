// tile_jit.h -- NVRTC-compiled, circuit-specialised tile kernels (tile_jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "tile_abi.h"

namespace qj {

// Returns the CUfunction of the specialised kernel for this lowered pass
// (compiling and caching it on first use), or nullptr with *err set when the
// JIT is unavailable or disabled (QJ_JIT=0).  *compile_ms is set on a compile.
template <typename R>
void* tile_jit_function(const TileArgs<R>& a, const void* mats_host, std::string* err, double* compile_ms);

cudaError_t tile_jit_launch(void* f, const void* args, unsigned grid, size_t smem, cudaStream_t st);

}  // namespace qj
