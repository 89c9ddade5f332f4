// small.h -- whole-state pass for states that fit one SM's shared memory
// (complex128 n <= 13, complex64 n <= 14: <= 128 KiB).  One CTA loads the
// state into SMEM once, applies a program of planned passes (the same
// per-gate Pass records the single-gate kernels take) with a block barrier
// between them, and stores it once: a whole circuit is ONE launch and one
// HBM round trip.  This is the regime of the paper's 10-qubit benchmarks
// (Table 1's small circuits), where per-gate launch latency,
// not bandwidth, is the cost.
#pragma once
#include <stdint.h>
#include <vector>
#include "qj_internal.h"

namespace qj {

constexpr int kSmallMaxC128 = 13;
constexpr int kSmallMaxC64 = 14;
constexpr int kSmallMaxK = 4;  // dense targets per op in the small kernel

inline int small_max_qubits(int amp_bytes) { return amp_bytes == 16 ? kSmallMaxC128 : kSmallMaxC64; }

// Whether the small kernel executes this pass.
bool small_supports(const Pass& p);

// A lowered program with a persistent device buffer (op records + data).
struct PreparedSmall {
    void* dev = nullptr;
    uint32_t nchunks = 0;  // program chunks (<= 16 KiB of op records + coefficients each)
    int nl = 0;
    int amp_bytes = 16;
    void* psi = nullptr;
};

template <typename R>
cudaError_t small_prepare(const std::vector<Pass>& prog, void* psi, int nl, PreparedSmall& out);
cudaError_t small_launch(const PreparedSmall& p, cudaStream_t st, LaunchStats& ls);
void small_release(PreparedSmall& p);
// One-shot: lower, upload (stream-ordered), launch, free.
template <typename R>
cudaError_t run_small(const std::vector<Pass>& prog, void* psi, int nl, cudaStream_t st, LaunchStats& ls);

}  // namespace qj
