// qj_internal.h -- host-side types shared by the C-ABI layer, the planner and
// the kernel launchers of libqj (never exposed through include/qj.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <complex>
#include <string>
#include <vector>

#include "../../include/qj.h"

namespace qj {

using cd = std::complex<double>;

// One planned pass over ONE shard.  Bit positions are PHYSICAL positions of
// the shard's local index (0 = least significant).
enum PassKind {
    PK_DENSE = 0,  // 2^k x 2^k matrix on k targets (Eq. 1), member `touch` mask
    PK_X = 1,      // X on 1 target: swap pairs (no arithmetic)
    PK_SWAP = 2,   // SWAP on 2 targets: exchange the |01>,|10> members
    PK_DIAG = 3,   // psi_i <- diag[row(i)] psi_i over k targets
    PK_PHASE = 4,  // psi_i <- phase * psi_i on the subspace fixed by `fix`
    PK_NEG = 5,    // psi_i <- -psi_i on the subspace fixed by `fix` (Z, CZ, ...)
};

struct Pass {
    int kind = PK_DENSE;
    int k = 0;                 // number of targets (DENSE/X/SWAP/DIAG)
    int tpos[QJ_MAX_TARGETS];  // target bit positions, listed (= matrix) order
    int nfix = 0;              // positions whose bit value is fixed (controls, phase pattern)
    int fpos[64];
    int fval[64];
    uint32_t touch = 0xffffffffu;  // DENSE: member mask over the listed-order member index
    std::vector<cd> m;             // DENSE: 4^k row-major; DIAG: 2^k; PHASE: 1
};

// Streaming multiprocessors of the current device (148 on B200); grids are
// sized in multiples of it.
inline int device_sms() {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        sms <= 0)
        return 148;
    return sms;
}

struct LaunchStats {
    uint64_t launches = 0;
};

// Algorithmic HBM bytes of a pass on a shard of 2^nl amplitudes of `bytes_per_amp`
// (C15: 2 * s * number of amplitudes the pass must change).
double pass_alg_bytes(const Pass& p, int nl, int bytes_per_amp);

// Launchers (kernels_*.cu).  R = float (complex64) or double (complex128).
template <typename R>
cudaError_t run_pass(const Pass& p, void* psi, int nl, cudaStream_t st, void* scratch,
                     size_t scratch_bytes, LaunchStats& ls);
template <typename R>
cudaError_t run_init(void* psi, int nl, uint64_t basis_local, bool set_one, cudaStream_t st,
                     LaunchStats& ls);
// probabilities of one shard: full (nq < 0, out = R[2^nl]) or marginal
// accumulated (fp64 atomics) into bins[2^nq]; positions = physical bits
// (pos < 0 means a global bit with value given by gbits).
template <typename R>
cudaError_t run_prob_full(const void* psi, int nl, void* out, cudaStream_t st, LaunchStats& ls);
template <typename R>
cudaError_t run_prob_marginal(const void* psi, int nl, const int* pos, const int* gval, int nq,
                              double* bins, cudaStream_t st, LaunchStats& ls);
template <typename R>
cudaError_t run_bins_to_out(const double* bins, uint64_t nbins, void* out, cudaStream_t st,
                            LaunchStats& ls);
template <typename R>
cudaError_t run_prob_scatter(const void* psi, int nl, uint64_t shard, int n, const int* cpos, void* out,
                             cudaStream_t st, LaunchStats& ls);
template <typename R>
cudaError_t run_exchange(void* a, void* b, int nl, int L, cudaStream_t st, LaunchStats& ls);

// measurement (measure.cu): consistent-subspace norm (fp64, deterministic
// order: partial[kNormBlocks] then *out), collapse write pass, samplers.
template <typename R>
cudaError_t run_subspace_norm(const void* psi, int nl, const int* pos, const int* val, int m, double* partial,
                              double* out, cudaStream_t st, LaunchStats& ls);
template <typename R>
cudaError_t run_collapse_apply(void* psi, int nl, uint64_t mask, uint64_t want, double scale, cudaStream_t st,
                               LaunchStats& ls);
size_t direct_scratch_bytes(uint64_t nbins);
constexpr uint64_t kTotalOverflow = ~0ull;  // direct sampler: weights sum to >= 15.5 (the 2^-60 CDF would wrap)
cudaError_t run_direct_cdf(const double* p, uint64_t nbins, void* scratch, cudaStream_t st, LaunchStats& ls);
const uint64_t* direct_total_ptr(const void* scratch, uint64_t nbins);
cudaError_t run_direct_shots(const void* scratch, uint64_t nbins, uint64_t nshots, uint64_t seed, int64_t* samples,
                             uint64_t* counts, cudaStream_t st, LaunchStats& ls);
cudaError_t run_metropolis(const double* p, int m, uint64_t nshots, uint64_t seed, uint32_t nchains, uint64_t burnin,
                           bool flip, int64_t* samples, uint64_t* counts, cudaStream_t st, LaunchStats& ls);
}  // namespace qj
