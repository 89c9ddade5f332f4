// tile_jit.h -- NVRTC-compiled, circuit-specialised tile kernels (tile_jit.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "tile_abi.h"

namespace qj {

#include <vector>

// A compiled, circuit-specialised tile kernel and what its launch needs:
// uniform coefficient slot j of TileArgs::uc takes fac[uc_src[j]] (>= 0) or
// mats[-uc_src[j] - 1]; `npt` per-thread factor tables are staged in SMEM by
// the kernel itself (launch with smem_extra more dynamic shared memory).
struct JitKernel {
    void* f = nullptr;
    std::vector<int32_t> uc_src;
    int npt = 0;
    size_t smem_extra = 0;
    int blocks = 2;  // resident CTAs per SM it was compiled for (grid = SMs x blocks)
    int threads = TILE_THREADS;  // block size (ring form: two workers)
    bool tmap = false;           // ring form with TMA tensor loads: TileArgs::tmap must be encoded
    bool l2_256 = false;         // ... with 256-byte L2 promotion (sibling-pair tile order)
};

// Checked JIT kernels (QJ_JIT_CHECK=1): the device flag their bounds checks
// set (nullptr when off), and whether it was set since the last call (resets it).
unsigned int* tile_check_flag();
bool tile_check_failed();

// Encode the ring form's tensor map (TileArgs::tmap) for a->psi.
template <typename R>
cudaError_t tile_jit_encode_tmap(TileArgs<R>* a, bool l2_256 = false);

// The specialised kernel for this lowered pass (compiled and cached on first
// use; `blob` is the host copy of the pass's program buffer), or nullptr with
// *err set when the JIT is unavailable or disabled (QJ_JIT=0).
template <typename R>
const JitKernel* tile_jit_kernel(const TileArgs<R>& a, const unsigned char* blob, std::string* err,
                                 double* compile_ms);

// Copy the kernel's uniform coefficients from the host program buffer into a->uc.
template <typename R>
void tile_jit_fill(const JitKernel& k, TileArgs<R>* a, const unsigned char* blob);

// Whether JIT kernels can be built here (NVRTC + driver found, QJ_JIT != 0).
bool tile_jit_available();

cudaError_t tile_jit_launch(void* f, const void* args, unsigned grid, size_t smem, cudaStream_t st,
                            int threads = TILE_THREADS);

}  // namespace qj
