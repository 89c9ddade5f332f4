// measure.cu -- measurement kernels (PAPER.md:239-242:
// "a custom operator for collapsing and re-normalizing states and a method for
// sampling shot frequencies based on Metropolis algorithm").
//
//   collapse   : P = sum |a|^2 over the consistent subspace only (reads 2^(n-m)
//                amplitudes, fixed grid + fixed-order reduction: deterministic),
//                then one pass writing a/sqrt(P) or 0 (reads only consistent
//                vectors).  DESIGN.md R26.
//   direct     : inverse CDF in 2^-60 fixed point -- exact uint64 prefix sums
//                (3-phase tile scan), per-shot binary search.  DESIGN.md R27.
//   Metropolis : one thread per independent chain, Philox4x32-10 counters
//                (t, chain, 1, 0), uniform or single-bit-flip proposals.  R28.
// Counts are warp-aggregated (__match_any_sync) before the global atomics.
#include <algorithm>

#include "common.cuh"
#include "philox.cuh"
#include "qj_internal.h"

namespace qj {
namespace {

constexpr int kMT = 256;
constexpr unsigned kNormBlocks = 1184;  // fixed (8 x 148): the reduction order never changes
constexpr int kScanTile = 4096;         // elements per scan tile (256 threads x 16)

__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < kMT / 32; ++i) t += red[i];
    return t;  // valid in thread 0
}

struct SubspaceArgs {
    uint64_t count;  // amplitudes in the consistent subspace of the shard
    int nins;
    int ins[64];     // measured local positions, ascending
    uint64_t want;   // their required values, as a bit pattern
};

template <typename R>
__global__ void __launch_bounds__(kMT) subspace_norm_kernel(const __grid_constant__ SubspaceArgs a, const void* p,
                                                            double* partial) {
    __shared__ double red[kMT / 32];
    const Cx<R>* psi = reinterpret_cast<const Cx<R>*>(p);
    double acc = 0.0;
    for (uint64_t j = (uint64_t)blockIdx.x * kMT + threadIdx.x; j < a.count; j += (uint64_t)gridDim.x * kMT) {
        uint64_t i = j;
        for (int k = 0; k < a.nins; ++k) i = insert_zero(i, a.ins[k]);
        const Cx<R> v = load_amp(psi, i | a.want);
        acc += (double)v.re * (double)v.re + (double)v.im * (double)v.im;
    }
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kMT) sum_partials_kernel(const double* partial, int np, double* out) {
    __shared__ double red[kMT / 32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < np; i += kMT) acc += partial[i];
    const double t = block_sum(acc, red);
    if (threadIdx.x == 0) *out = t;
}

template <typename R>
__global__ void __launch_bounds__(kMT) collapse_apply_kernel(void* p, uint64_t nvec, uint64_t mask, uint64_t want,
                                                             R scale) {
    using Vec = typename VecT<R>::type;
    constexpr int V = VecT<R>::V;
    Vec* psi = reinterpret_cast<Vec*>(p);
    const Vec zv = {};
    for (uint64_t i = (uint64_t)blockIdx.x * kMT + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * kMT) {
        bool keep[1 << V], any = false;
#pragma unroll
        for (int w = 0; w < (1 << V); ++w) {
            keep[w] = ((((i << V) | (uint64_t)w) & mask) == want);
            any |= keep[w];
        }
        if (!any) {
            stv(psi + i, zv);
            continue;
        }
        Cx<R> amp[1 << V];
        unpack(ldv(psi + i), amp);
#pragma unroll
        for (int w = 0; w < (1 << V); ++w)
            amp[w] = keep[w] ? Cx<R>{amp[w].re * scale, amp[w].im * scale} : Cx<R>{R(0), R(0)};
        stv(psi + i, pack(amp));
    }
}

// tiny shards (fewer amplitudes than one vector): scalar
template <typename R>
__global__ void collapse_apply_scalar_kernel(void* p, uint64_t namp, uint64_t mask, uint64_t want, R scale) {
    Cx<R>* psi = reinterpret_cast<Cx<R>*>(p);
    for (uint64_t i = threadIdx.x; i < namp; i += blockDim.x) {
        const Cx<R> v = psi[i];
        psi[i] = ((i & mask) == want) ? Cx<R>{v.re * scale, v.im * scale} : Cx<R>{R(0), R(0)};
    }
}

// ---------------------------------------------------------------- fixed-point scan
__device__ __forceinline__ uint64_t fixq(double p) {
    // rint(p * 2^60); negative and NaN -> 0 (R27)
    return (p > 0.0) ? __double2ull_rn(p * 0x1.0p60) : 0ull;
}
__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }  // 16 doubles per bank row

// Inclusive scan of one tile of q values held in smem; returns the tile total
// (thread 0) and leaves the inclusive prefix in smem.
__device__ uint64_t tile_scan(const double* p, uint64_t nb, uint64_t tile, uint64_t* s, uint64_t* wsum) {
    const uint64_t base = tile * kScanTile;
    for (int i = threadIdx.x; i < kScanTile; i += kMT) {
        const uint64_t k = base + i;
        s[spad(i)] = k < nb ? fixq(p[k]) : 0ull;
    }
    __syncthreads();
    uint64_t v[16], run = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        run += s[spad(threadIdx.x * 16 + j)];
        v[j] = run;
    }
    // exclusive scan of thread totals: warp inclusive scan + warp totals
    const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t inc = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (l >= o) inc += t;
    }
    if (l == 31) wsum[w] = inc;
    __syncthreads();
    uint64_t wpre = 0;
    for (int i = 0; i < w; ++i) wpre += wsum[i];
    const uint64_t pre = wpre + inc - run;
#pragma unroll
    for (int j = 0; j < 16; ++j) s[spad(threadIdx.x * 16 + j)] = pre + v[j];
    uint64_t total = 0;
    for (int i = 0; i < kMT / 32; ++i) total += wsum[i];
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(kMT) scan_tiles_kernel(const double* p, uint64_t nb, uint64_t* tile_tot,
                                                         double* tile_dsum) {
    __shared__ uint64_t s[kScanTile + kScanTile / 16];
    __shared__ uint64_t wsum[kMT / 32];
    __shared__ double dsum[kMT / 32];
    // fp64 weight of the tile, only to reject totals the 2^-60 fixed point cannot hold
    double d = 0.0;
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
    for (int i = threadIdx.x; i < kScanTile; i += kMT)
        if (base + i < nb && p[base + i] > 0.0) d += p[base + i];
#pragma unroll
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) dsum[threadIdx.x >> 5] = d;
    const uint64_t t = tile_scan(p, nb, blockIdx.x, s, wsum);  // (its barriers order dsum)
    if (threadIdx.x == 0) {
        double e = 0.0;
        for (int i = 0; i < kMT / 32; ++i) e += dsum[i];
        tile_tot[blockIdx.x] = t;
        tile_dsum[blockIdx.x] = e;
    }
}

// exclusive scan of the tile totals in place (one block), total -> *total
__global__ void __launch_bounds__(1024) scan_offsets_kernel(uint64_t* tot, const double* dsum, uint64_t ntiles,
                                                            uint64_t* total) {
    __shared__ uint64_t part[1024];
    __shared__ double dpart[1024];
    const uint64_t per = (ntiles + 1023) / 1024;
    const uint64_t b = threadIdx.x * per, e = min(ntiles, b + per);
    uint64_t run = 0;
    double drun = 0.0;
    for (uint64_t i = b; i < e; ++i) {
        run += tot[i];
        drun += dsum[i];
    }
    part[threadIdx.x] = run;
    dpart[threadIdx.x] = drun;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t acc = 0;
        double dacc = 0.0;
        for (int i = 0; i < 1024; ++i) {
            const uint64_t x = part[i];
            part[i] = acc;
            acc += x;
            dacc += dpart[i];
        }
        // the fixed-point CDF holds totals below 2^64 = 16 * 2^60: larger
        // weights would wrap; flag them for the host check (kTotalOverflow)
        *total = (dacc >= 15.5 || !(dacc == dacc)) ? kTotalOverflow : acc;
    }
    __syncthreads();
    uint64_t acc = part[threadIdx.x];
    for (uint64_t i = b; i < e; ++i) {
        const uint64_t x = tot[i];
        tot[i] = acc;
        acc += x;
    }
}

__global__ void __launch_bounds__(kMT) scan_write_kernel(const double* p, uint64_t nb, const uint64_t* off,
                                                         uint64_t* cdf) {
    __shared__ uint64_t s[kScanTile + kScanTile / 16];
    __shared__ uint64_t wsum[kMT / 32];
    tile_scan(p, nb, blockIdx.x, s, wsum);
    const uint64_t base = (uint64_t)blockIdx.x * kScanTile, o = off[blockIdx.x];
    for (int i = threadIdx.x; i < kScanTile; i += kMT)
        if (base + i < nb) cdf[base + i] = o + s[spad(i)];
}

__device__ __forceinline__ void record(uint64_t k, uint64_t slot, int64_t* samples, unsigned long long* counts) {
    if (samples) samples[slot] = (int64_t)k;
    if (counts) {
        const unsigned act = __activemask();
        const unsigned peers = __match_any_sync(act, k);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + k, (unsigned long long)__popc(peers));
    }
}

__global__ void __launch_bounds__(kMT) direct_shots_kernel(const uint64_t* cdf, uint64_t nb, const uint64_t* total,
                                                           uint64_t nshots, uint32_t k0, uint32_t k1,
                                                           int64_t* samples, unsigned long long* counts) {
    const uint64_t Q = *total;
    for (uint64_t i = (uint64_t)blockIdx.x * kMT + threadIdx.x; i < nshots; i += (uint64_t)gridDim.x * kMT) {
        const U4 w = philox4x32_10(U4{(uint32_t)i, (uint32_t)(i >> 32), RNG_STREAM_DIRECT, 0u}, k0, k1);
        const uint64_t r = ((((uint64_t)w.x) << 32) | w.y) >> 11;  // 53 bits
        const uint64_t v = __umul64hi(r << 11, Q);                // floor(r Q / 2^53)
        uint64_t lo = 0, hi = nb - 1;                             // first k with cdf[k] > v
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (__ldg(cdf + mid) > v) hi = mid;
            else lo = mid + 1;
        }
        record(lo, i, samples, counts);
    }
}

struct ChainArgs {
    const double* p;
    uint64_t mask;
    int m;
    int flip;
    uint32_t nchains;
    uint64_t base, extra;  // chain c records base + (c < extra) shots
    uint64_t burnin;
    uint32_t k0, k1;
    int64_t* samples;
    unsigned long long* counts;
};

__global__ void __launch_bounds__(kMT) metropolis_kernel(const __grid_constant__ ChainArgs a) {
    const uint32_t c = blockIdx.x * kMT + threadIdx.x;
    if (c >= a.nchains) return;
    const uint64_t shots = a.base + (c < a.extra ? 1 : 0);
    const uint64_t off = (uint64_t)c * a.base + min((uint64_t)c, a.extra);
    U4 w = philox4x32_10(U4{0xFFFFFFFFu, c, RNG_STREAM_METROPOLIS, 0u}, a.k0, a.k1);
    uint64_t x = ((((uint64_t)w.x) << 32) | w.y) & a.mask;
    double px = __ldg(a.p + x);
    const uint64_t steps = a.burnin + shots;
    for (uint64_t t = 0; t < steps; ++t) {
        w = philox4x32_10(U4{(uint32_t)t, c, RNG_STREAM_METROPOLIS, 0u}, a.k0, a.k1);
        const uint64_t y = a.flip ? (x ^ (1ull << (w.x % (uint32_t)(a.m > 0 ? a.m : 1)))) & a.mask
                                  : ((((uint64_t)w.x) << 32) | w.y) & a.mask;
        const double py = __ldg(a.p + y);
        const double u = u53(w.z, w.w);
        if (px == 0.0 || u * px < py) {
            x = y;
            px = py;
        }
        if (t >= a.burnin) record(x, off + (t - a.burnin), a.samples, a.counts);
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers
template <typename R>
cudaError_t run_subspace_norm(const void* psi, int nl, const int* pos, const int* val, int m, double* partial,
                              double* out, cudaStream_t st, LaunchStats& ls) {
    SubspaceArgs a{};
    a.nins = m;
    int sorted[64];
    for (int i = 0; i < m; ++i) sorted[i] = pos[i];
    std::sort(sorted, sorted + m);
    for (int i = 0; i < m; ++i) a.ins[i] = sorted[i];
    a.want = 0;
    for (int i = 0; i < m; ++i)
        if (val[i]) a.want |= 1ull << pos[i];
    a.count = 1ull << (nl - m);
    const uint64_t blocks = std::min<uint64_t>(kNormBlocks, (a.count + kMT - 1) / kMT);
    subspace_norm_kernel<R><<<(unsigned)blocks, kMT, 0, st>>>(a, psi, partial);
    sum_partials_kernel<<<1, kMT, 0, st>>>(partial, (int)blocks, out);
    ls.launches += 2;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_collapse_apply(void* psi, int nl, uint64_t mask, uint64_t want, double scale, cudaStream_t st,
                               LaunchStats& ls) {
    constexpr int V = VecT<R>::V;
    if (nl < V) {
        collapse_apply_scalar_kernel<R><<<1, 32, 0, st>>>(psi, 1ull << nl, mask, want, (R)scale);
    } else {
        const uint64_t nvec = 1ull << (nl - V);
        const uint64_t blocks = std::min<uint64_t>(148ull * 16, (nvec + kMT - 1) / kMT);
        collapse_apply_kernel<R><<<(unsigned)blocks, kMT, 0, st>>>(psi, nvec, mask, want, (R)scale);
    }
    ls.launches++;
    return cudaGetLastError();
}

size_t direct_scratch_bytes(uint64_t nb) {
    const uint64_t ntiles = (nb + kScanTile - 1) / kScanTile;
    return (nb + ntiles + 1) * sizeof(uint64_t) + ntiles * sizeof(double);
}

cudaError_t run_direct_cdf(const double* p, uint64_t nb, void* scratch, cudaStream_t st, LaunchStats& ls) {
    const uint64_t ntiles = (nb + kScanTile - 1) / kScanTile;
    uint64_t* cdf = static_cast<uint64_t*>(scratch);
    uint64_t* tot = cdf + nb;
    uint64_t* total = tot + ntiles;
    double* dsum = reinterpret_cast<double*>(total + 1);
    scan_tiles_kernel<<<(unsigned)ntiles, kMT, 0, st>>>(p, nb, tot, dsum);
    scan_offsets_kernel<<<1, 1024, 0, st>>>(tot, dsum, ntiles, total);
    scan_write_kernel<<<(unsigned)ntiles, kMT, 0, st>>>(p, nb, tot, cdf);
    ls.launches += 3;
    return cudaGetLastError();
}

const uint64_t* direct_total_ptr(const void* scratch, uint64_t nb) {
    const uint64_t ntiles = (nb + kScanTile - 1) / kScanTile;
    return static_cast<const uint64_t*>(scratch) + nb + ntiles;
}

cudaError_t run_direct_shots(const void* scratch, uint64_t nb, uint64_t nshots, uint64_t seed, int64_t* samples,
                             uint64_t* counts, cudaStream_t st, LaunchStats& ls) {
    const uint64_t* cdf = static_cast<const uint64_t*>(scratch);
    const uint64_t blocks = std::min<uint64_t>(148ull * 16, (nshots + kMT - 1) / kMT);
    direct_shots_kernel<<<(unsigned)blocks, kMT, 0, st>>>(cdf, nb, direct_total_ptr(scratch, nb), nshots,
                                                          (uint32_t)seed, (uint32_t)(seed >> 32), samples,
                                                          reinterpret_cast<unsigned long long*>(counts));
    ls.launches++;
    return cudaGetLastError();
}

cudaError_t run_metropolis(const double* p, int m, uint64_t nshots, uint64_t seed, uint32_t nchains, uint64_t burnin,
                           bool flip, int64_t* samples, uint64_t* counts, cudaStream_t st, LaunchStats& ls) {
    ChainArgs a{};
    a.p = p;
    a.m = m;
    a.mask = (m >= 64) ? ~0ull : ((1ull << m) - 1);
    a.flip = flip ? 1 : 0;
    a.nchains = nchains;
    a.base = nshots / nchains;
    a.extra = nshots % nchains;
    a.burnin = burnin;
    a.k0 = (uint32_t)seed;
    a.k1 = (uint32_t)(seed >> 32);
    a.samples = samples;
    a.counts = reinterpret_cast<unsigned long long*>(counts);
    metropolis_kernel<<<(nchains + kMT - 1) / kMT, kMT, 0, st>>>(a);
    ls.launches++;
    return cudaGetLastError();
}

#define QJ_INST_MEASURE(R)                                                                                   \
    template cudaError_t run_subspace_norm<R>(const void*, int, const int*, const int*, int, double*, double*, \
                                              cudaStream_t, LaunchStats&);                                     \
    template cudaError_t run_collapse_apply<R>(void*, int, uint64_t, uint64_t, double, cudaStream_t, LaunchStats&);
QJ_INST_MEASURE(float)
QJ_INST_MEASURE(double)

}  // namespace qj
