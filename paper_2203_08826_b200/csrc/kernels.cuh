// kernels.cuh -- sm_100a single-gate pass kernels of libqj and their host
// launchers.  Instantiated for float (complex64) in kernels_c64.cu and for
// double (complex128) in kernels_c128.cu.
//
// What each pass computes is Eq. 1 restricted to the index
// groups a gate touches.  Groups are enumerated by bit insertion
// (PAPER.md:221-227 listing), never from stored index tables.
//
// gate_warp_kernel -- the workhorse (dense k<=5 matrices, X, SWAP, fSim).
//   * A warp owns a "unit": 32 consecutive 16-byte vectors (512 B, fully
//     coalesced 128-bit loads/stores).  Bits [0, LB) of the amplitude index are
//     vector (c64 bit 0) + lane bits; bits >= LB are outer bits.
//   * Outer targets (H of them) become a register dimension: each lane loads
//     its vector at base | pattern for every 2^H outer pattern.
//   * Lane targets (KL of them, bits V..V+4) are exchanged with warp shuffles:
//     the lane fetches its partners' registers with shfl.xor, so the gate's
//     2^k inputs are in registers without any shared-memory round trip.
//   * A vector target (c64 bit 0, KV = 1) is already inside the thread.
//   * Outer controls / fixed bits are removed from the enumeration by bit
//     insertion (only touched amplitudes are read: the sparsity of controlled
//     gates); low controls predicate loads and stores.
//   The host permutes the matrix into the canonical bit order
//   [outer targets | vector target | lane targets] so every register index is
//   a compile-time constant; the lane-dependent part of the row/column index
//   (ell) is folded in by conjugating the matrix with ell (G[a^ell][b^ell]).
// gate_simple_kernel -- tiny states (fewer than one warp unit): one thread per
//   group, the paper's literal kernel shape.
// gate_bigk_kernel -- 6..8 targets: one block per group, staged in SMEM.
// diag_kernel -- diagonal gates, phases, sign flips: no exchange at all.
#pragma once

#include <algorithm>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "common.cuh"
#include "dense_tc.h"
#include "qj_internal.h"

namespace qj {

constexpr int kThreads = 256;

// ---------------------------------------------------------------- geometry
struct WarpGeom {
    uint64_t units;     // number of warp units
    uint64_t fix_val;   // values OR-ed in at outer fixed positions
    uint32_t low_mask;  // low-bit (vector + lane) fixed positions ...
    uint32_t low_val;   // ... and their required values
    uint32_t touch;     // canonical member mask
    int nins;           // outer positions removed from the enumeration (ascending)
    int ins_pos[MAXB];
    int h_pos[5];       // outer target positions, canonical order
    int l_pos[5];       // lane target positions, canonical order
};

template <typename R, int K>
struct WarpArgs {
    WarpGeom g;
    void* psi;
    Cx<R> m[1 << K][1 << K];  // canonical order
};

__device__ __forceinline__ uint64_t unit_base(uint64_t u, int lb, int nins, const int* ins_pos,
                                              uint64_t fix_val) {
    uint64_t x = u << lb;
    for (int i = 0; i < nins; ++i) x = insert_zero(x, ins_pos[i]);
    return x | fix_val;
}

// MODE 0: dense matrix; 1: X (swap the two members); 2: SWAP (exchange 01 <-> 10)
template <typename R, int K, int H, int KV, int MODE>
__global__ void __launch_bounds__(kThreads) gate_warp_kernel(const __grid_constant__ WarpArgs<R, K> a) {
    using Vec = typename VecT<R>::type;
    constexpr int V = VecT<R>::V;
    constexpr int LB = V + 5;
    constexpr int KL = K - H - KV;
    static_assert(KL >= 0 && KL <= 5, "bad split");
    constexpr int NW = 1 << V, NP = 1 << H, NM = 1 << KL, D = 1 << K;
    constexpr int U = (H + V >= 2) ? 1 : (1 << (2 - H - V));
    constexpr bool SMEM_M = (MODE == 0) && (K >= 3);
    constexpr bool PRE = (MODE == 0) && (K <= 2);
    constexpr int NG = KV ? 1 : NW;           // independent groups per thread per unit
    constexpr int NR = NP * (KV ? NW : 1);    // own rows per group
    constexpr bool EAGER = (V == 0) || (H >= 4);

    __shared__ Cx<R> sm[SMEM_M ? D * D : 1];
    if constexpr (SMEM_M) {
        const Cx<R>* src = &a.m[0][0];
        for (int i = threadIdx.x; i < D * D; i += blockDim.x) sm[i] = src[i];
        __syncthreads();
    }

    const int lane = threadIdx.x & 31;
    const uint32_t lowlane = (uint32_t)lane << V;
    int ell = 0;
#pragma unroll
    for (int i = 0; i < KL; ++i) ell = (ell << 1) | ((lowlane >> a.g.l_pos[i]) & 1);
    int xm[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        int x = 0;
#pragma unroll
        for (int i = 0; i < KL; ++i)
            if ((m >> (KL - 1 - i)) & 1) x |= 1 << (a.g.l_pos[i] - V);
        xm[m] = x;
    }
    bool wact[NW];
    bool lane_any = false;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        wact[w] = ((lowlane | w) & a.g.low_mask) == a.g.low_val;
        lane_any |= wact[w];
    }
    // touched[p][w]: member index (canonical) of own register (p, w)
    bool tch[NP][NW];
    bool ld_p[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) {
        ld_p[p] = false;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const int mem = (p << (KV + KL)) | ((KV ? w : 0) << KL) | ell;
            tch[p][w] = ((a.g.touch >> mem) & 1u) && wact[w];
            ld_p[p] |= tch[p][w];
        }
    }
    uint64_t hb[H > 0 ? H : 1];
#pragma unroll
    for (int i = 0; i < H; ++i) hb[i] = 1ull << a.g.h_pos[i];

    Cx<R> co[PRE ? NR : 1][PRE ? D : 1];
    if constexpr (PRE) {
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int p = KV ? (r >> 1) : r, wv = KV ? (r & 1) : 0;
            const int row = (p << (KV + KL)) | (wv << KL);
#pragma unroll
            for (int c = 0; c < D; ++c) co[r][c] = a.m[row ^ ell][c ^ ell];
        }
    }
    // SWAP with lane targets: conjugating P by ell flips both bits iff ell's
    // two canonical bits differ (P(a^ell)^ell = P(a) ^ (P(ell)^ell)).
    const int ell_par = __popc(ell) & 1;

    Vec* psi = reinterpret_cast<Vec*>(a.psi);
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const Vec zv = {};

    for (uint64_t u0 = gw * U; u0 < a.g.units; u0 += nwarps * U) {
        uint64_t base[U];
        Vec v[U][NP];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const uint64_t u = u0 + uu;
            base[uu] = unit_base(u, LB, a.g.nins, a.g.ins_pos, a.g.fix_val) | lowlane;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                uint64_t off = 0;
#pragma unroll
                for (int i = 0; i < H; ++i)
                    if ((p >> (H - 1 - i)) & 1) off |= hb[i];
                v[uu][p] = (u < a.g.units && ld_p[p]) ? ldv(psi + ((base[uu] | off) >> V)) : zv;
            }
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            if (u0 + uu >= a.g.units) break;  // warp-uniform
            Cx<R> amp[NP][NW];
#pragma unroll
            for (int p = 0; p < NP; ++p) unpack(v[uu][p], amp[p]);
            Cx<R> X[NM][NP][NW];
#pragma unroll
            for (int p = 0; p < NP; ++p)
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    X[0][p][w] = amp[p][w];
#pragma unroll
                    for (int m = 1; m < NM; ++m) X[m][p][w] = shfl_xor(amp[p][w], xm[m]);
                }
            Cx<R> res[EAGER ? 1 : NP][NW];
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                Cx<R> in[D];
#pragma unroll
                for (int p = 0; p < NP; ++p)
#pragma unroll
                    for (int wv = 0; wv < (KV ? NW : 1); ++wv)
#pragma unroll
                        for (int m = 0; m < NM; ++m)
                            in[(p << (KV + KL)) | (wv << KL) | m] = X[m][p][KV ? wv : g];
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const int p = KV ? (r >> 1) : r, wv = KV ? (r & 1) : 0;
                    const int w = KV ? wv : g;
                    const int row = (p << (KV + KL)) | (wv << KL);
                    Cx<R> o;
                    if constexpr (MODE == 0) {
                        o = Cx<R>{R(0), R(0)};
#pragma unroll
                        for (int c = 0; c < D; ++c) {
                            Cx<R> coef;
                            if constexpr (PRE) coef = co[r][c];
                            else if constexpr (SMEM_M) coef = sm[(row ^ ell) * D + (c ^ ell)];
                            else coef = a.m[row ^ ell][c ^ ell];
                            cfma(o, coef, in[c]);
                        }
                    } else if constexpr (MODE == 1) {
                        o = in[row ^ 1];
                    } else {
                        // canonical 2-bit index b1 b0; P swaps the bits
                        const int pr = ((row & 1) << 1) | ((row >> 1) & 1);
                        o = ell_par ? in[pr ^ 3] : in[pr];
                    }
                    if (!tch[p][w]) o = amp[p][w];
                    if constexpr (EAGER) {
                        if (tch[p][w]) {
                            uint64_t off = 0;
#pragma unroll
                            for (int i = 0; i < H; ++i)
                                if ((p >> (H - 1 - i)) & 1) off |= hb[i];
                            const uint64_t idx = base[uu] | off | (uint64_t)w;
                            store_amp(a.psi, idx, o);
                        }
                    } else {
                        res[p][w] = o;
                    }
                }
            }
            if constexpr (!EAGER) {
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    if (!ld_p[p]) continue;
                    uint64_t off = 0;
#pragma unroll
                    for (int i = 0; i < H; ++i)
                        if ((p >> (H - 1 - i)) & 1) off |= hb[i];
                    stv(psi + ((base[uu] | off) >> V), pack(res[p]));
                }
            }
        }
    }
}

// ------------------------------------------------------------ simple kernel
struct SimpleGeom {
    uint64_t groups;
    uint64_t fix_val;
    uint32_t touch;
    int nins;
    int ins_pos[MAXB];
    int tpos[5];
};
template <typename R, int K>
struct SimpleArgs {
    SimpleGeom g;
    void* psi;
    Cx<R> m[1 << K][1 << K];  // listed order
};

template <typename R, int K>
__global__ void __launch_bounds__(kThreads) gate_simple_kernel(const __grid_constant__ SimpleArgs<R, K> a) {
    constexpr int D = 1 << K;
    Cx<R>* psi = reinterpret_cast<Cx<R>*>(a.psi);
    for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < a.g.groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = g;
        for (int i = 0; i < a.g.nins; ++i) base = insert_zero(base, a.g.ins_pos[i]);
        base |= a.g.fix_val;
        uint64_t idx[D];
        Cx<R> in[D];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            uint64_t x = base;
#pragma unroll
            for (int i = 0; i < K; ++i)
                if ((j >> (K - 1 - i)) & 1) x |= 1ull << a.g.tpos[i];
            idx[j] = x;
            in[j] = ((a.g.touch >> j) & 1u) ? psi[x] : Cx<R>{R(0), R(0)};
        }
#pragma unroll
        for (int r = 0; r < D; ++r) {
            if (!((a.g.touch >> r) & 1u)) continue;
            Cx<R> o{R(0), R(0)};
#pragma unroll
            for (int c = 0; c < D; ++c) cfma(o, a.m[r][c], in[c]);
            psi[idx[r]] = o;
        }
    }
}

// ------------------------------------------------------------ big-k kernel
// 6..8 targets: one block of 2^k threads per group; the group is gathered
// into SMEM, each thread computes one output row (matrix read from global /
// L2), then scatters.  Rare in practice (the fast path is k <= 5).
struct BigKArgs {
    uint64_t groups;
    uint64_t fix_val;
    int k;
    int nins;
    int ins_pos[MAXB];
    int tpos[QJ_MAX_TARGETS];
    void* psi;
    const void* m;  // device, listed order, D*D
};

template <typename R>
__global__ void gate_bigk_kernel(const __grid_constant__ BigKArgs a) {
    __shared__ Cx<R> sv[1 << QJ_MAX_TARGETS];
    const int D = 1 << a.k;
    const int j = threadIdx.x;
    const Cx<R>* M = reinterpret_cast<const Cx<R>*>(a.m);
    Cx<R>* psi = reinterpret_cast<Cx<R>*>(a.psi);
    for (uint64_t g = blockIdx.x; g < a.groups; g += gridDim.x) {
        uint64_t x = g;
        for (int i = 0; i < a.nins; ++i) x = insert_zero(x, a.ins_pos[i]);
        x |= a.fix_val;
        for (int i = 0; i < a.k; ++i)
            if ((j >> (a.k - 1 - i)) & 1) x |= 1ull << a.tpos[i];
        sv[j] = psi[x];
        __syncthreads();
        Cx<R> o{R(0), R(0)};
        for (int c = 0; c < D; ++c) cfma(o, M[(size_t)j * D + c], sv[c]);
        psi[x] = o;
        __syncthreads();
    }
}

// ------------------------------------------------------------ diagonal kernel
// MODE 0: psi_i <- table[row(i)] psi_i (row from the target bits, listed order)
// MODE 1: psi_i <- phase psi_i on the subspace fixed by the inserted bits
// MODE 2: psi_i <- -psi_i  on that subspace (exact sign flip: Z, CZ, CCZ ...)
template <typename R>
struct DiagArgs {
    uint64_t units;
    uint64_t fix_val;
    uint32_t low_mask, low_val;
    int nins;
    int ins_pos[MAXB];
    int nt;
    int tpos[QJ_MAX_TARGETS];
    void* psi;
    Cx<R> phase;
    Cx<R> table[1 << QJ_MAX_TARGETS];
};

template <typename R, int MODE>
__global__ void __launch_bounds__(kThreads) diag_kernel(const __grid_constant__ DiagArgs<R> a) {
    using Vec = typename VecT<R>::type;
    constexpr int V = VecT<R>::V;
    constexpr int LB = V + 5;
    constexpr int NW = 1 << V;
    constexpr int U = 4;
    __shared__ Cx<R> tab[MODE == 0 ? (1 << QJ_MAX_TARGETS) : 1];
    if constexpr (MODE == 0) {
        for (int i = threadIdx.x; i < (1 << a.nt); i += blockDim.x) tab[i] = a.table[i];
        __syncthreads();
    }
    const int lane = threadIdx.x & 31;
    const uint32_t lowlane = (uint32_t)lane << V;
    bool wact[NW];
    bool any = false;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
        wact[w] = ((lowlane | w) & a.low_mask) == a.low_val;
        any |= wact[w];
    }
    // (tried: lanes whose 32-byte sector partner is active also load and store
    // unchanged data, for whole-sector writes -- measured slower for CU1 on
    // bits (0,1) / (0,29), 6.5 -> 7.0 / 3.9 -> 5.0 ms; only touched vectors move)
    const bool io = any;
    Vec* psi = reinterpret_cast<Vec*>(a.psi);
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const Vec zv = {};
    for (uint64_t u0 = gw * U; u0 < a.units; u0 += nwarps * U) {
        uint64_t base[U];
        Vec v[U];
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            const uint64_t u = u0 + uu;
            base[uu] = unit_base(u, LB, a.nins, a.ins_pos, a.fix_val) | lowlane;
            v[uu] = (u < a.units && io) ? ldv(psi + (base[uu] >> V)) : zv;
        }
#pragma unroll
        for (int uu = 0; uu < U; ++uu) {
            if (u0 + uu >= a.units || !io) continue;
            Cx<R> amp[NW];
            unpack(v[uu], amp);
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                if (!wact[w]) continue;
                if constexpr (MODE == 0) {
                    const uint64_t idx = base[uu] | (uint64_t)w;
                    int row = 0;
                    for (int i = 0; i < a.nt; ++i) row = (row << 1) | (int)((idx >> a.tpos[i]) & 1u);
                    amp[w] = cmul(tab[row], amp[w]);
                } else if constexpr (MODE == 1) {
                    amp[w] = cmul(a.phase, amp[w]);
                } else {
                    amp[w] = Cx<R>{-amp[w].re, -amp[w].im};
                }
            }
            stv(psi + (base[uu] >> V), pack(amp));
        }
    }
}

// ------------------------------------------------------------ state init
template <typename R>
__global__ void __launch_bounds__(kThreads) init_kernel(void* p, uint64_t nvec, uint64_t basis, int set_one) {
    using Vec = typename VecT<R>::type;
    constexpr int V = VecT<R>::V;
    Vec* psi = reinterpret_cast<Vec*>(p);
    const Vec zv = {};
    const uint64_t bvec = basis >> V;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (set_one && i == bvec) {
            Cx<R> amp[1 << V];
#pragma unroll
            for (int w = 0; w < (1 << V); ++w)
                amp[w] = Cx<R>{(uint64_t)w == (basis & ((1u << V) - 1)) ? R(1) : R(0), R(0)};
            stv(psi + i, pack(amp));
        } else {
            stv(psi + i, zv);
        }
    }
}
// tiny states (fewer amplitudes than one vector holds): scalar init
template <typename R>
__global__ void init_scalar_kernel(void* p, uint64_t namp, uint64_t basis, int set_one) {
    Cx<R>* psi = reinterpret_cast<Cx<R>*>(p);
    for (uint64_t i = threadIdx.x; i < namp; i += blockDim.x)
        psi[i] = Cx<R>{(set_one && i == basis) ? R(1) : R(0), R(0)};
}

// ------------------------------------------------------------ probabilities
template <typename R>
__global__ void __launch_bounds__(kThreads) prob_full_kernel(const void* p, void* out, uint64_t namp) {
    const Cx<R>* psi = reinterpret_cast<const Cx<R>*>(p);
    R* o = reinterpret_cast<R*>(out);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < namp;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const Cx<R> a = psi[i];
        o[i] = a.re * a.re + a.im * a.im;
    }
}

struct MargArgs {
    uint64_t namp;
    int nq;
    int pos[64];      // physical local bit (>= 0) or -1: constant bit
    int cbit[64];     // value of a constant bit
    double* bins;     // 2^nq fp64 accumulators (global)
    const void* psi;
};

// Marginal fast path: every listed bit lies above the block's contiguous chunk
// of 2^cb amplitudes, so the whole chunk falls in one bin.  Vectorised loads,
// fp64 accumulation, block reduction, one atomic per chunk.
template <typename R>
__global__ void __launch_bounds__(kThreads) prob_chunk_kernel(const __grid_constant__ MargArgs a, int cb) {
    using Vec = typename VecT<R>::type;
    constexpr int V = VecT<R>::V;
    __shared__ double red[kThreads / 32];
    const Vec* psi = reinterpret_cast<const Vec*>(a.psi);
    const uint64_t chunk = blockIdx.x;
    const uint64_t nvec = 1ull << (cb - V);
    const uint64_t v0 = chunk * nvec;
    double acc0 = 0.0, acc1 = 0.0;
    uint64_t i = threadIdx.x;
    for (; i + kThreads < nvec; i += 2 * kThreads) {
        Cx<R> x[1 << V], y[1 << V];
        unpack(ldv(psi + v0 + i), x);
        unpack(ldv(psi + v0 + i + kThreads), y);
#pragma unroll
        for (int w = 0; w < (1 << V); ++w) {
            acc0 = fma((double)x[w].re, (double)x[w].re, fma((double)x[w].im, (double)x[w].im, acc0));
            acc1 = fma((double)y[w].re, (double)y[w].re, fma((double)y[w].im, (double)y[w].im, acc1));
        }
    }
    for (; i < nvec; i += kThreads) {
        Cx<R> x[1 << V];
        unpack(ldv(psi + v0 + i), x);
#pragma unroll
        for (int w = 0; w < (1 << V); ++w)
            acc0 = fma((double)x[w].re, (double)x[w].re, fma((double)x[w].im, (double)x[w].im, acc0));
    }
    double s = acc0 + acc1;
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) t += red[w];
        const uint64_t base = chunk << cb;
        uint32_t o = 0;
        for (int q = 0; q < a.nq; ++q) {
            const uint32_t b = a.pos[q] >= 0 ? (uint32_t)((base >> a.pos[q]) & 1u) : (uint32_t)a.cbit[q];
            o = (o << 1) | b;
        }
        atomicAdd(&a.bins[o], t);
    }
}

// Marginal probabilities, general case.  The output bin of index i is
// assembled from per-byte tables (bin bits contributed by each byte of i).
// Each thread keeps a running (bin, sum) and flushes it -- to SMEM bins
// (nq <= 12) or straight to the global fp64 bins -- only when its bin
// changes: with a grid stride that is a multiple of 2^(max listed bit + 1) a
// thread's bin never changes, and listed high bits change it rarely.
template <typename R, bool SMEM>
__global__ void __launch_bounds__(kThreads) prob_marg_kernel(const __grid_constant__ MargArgs a, int nbytes) {
    __shared__ double sb[SMEM ? 4096 : 1];
    __shared__ uint32_t tbl[8][256];
    const int nb = 1 << a.nq;
    if constexpr (SMEM) {
        for (int i = threadIdx.x; i < nb; i += blockDim.x) sb[i] = 0.0;
    }
    uint32_t cst = 0;  // constant (global) bits of the bin
    for (int q = 0; q < a.nq; ++q)
        if (a.pos[q] < 0 && a.cbit[q]) cst |= 1u << (a.nq - 1 - q);
    for (int e = threadIdx.x; e < nbytes * 256; e += blockDim.x) {
        const int c = e >> 8, v = e & 255;
        uint32_t o = c == 0 ? cst : 0u;
        for (int q = 0; q < a.nq; ++q) {
            const int p = a.pos[q] - 8 * c;
            if (a.pos[q] >= 0 && p >= 0 && p < 8 && ((v >> p) & 1)) o |= 1u << (a.nq - 1 - q);
        }
        tbl[c][v] = o;
    }
    __syncthreads();
    const Cx<R>* psi = reinterpret_cast<const Cx<R>*>(a.psi);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t cur = 0xffffffffu;
    double acc = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.namp; i += stride) {
        const Cx<R> v = psi[i];
        uint32_t o = 0;
        for (int c = 0; c < nbytes; ++c) o |= tbl[c][(i >> (8 * c)) & 255];
        if (o != cur) {
            if (cur != 0xffffffffu) {
                if constexpr (SMEM) atomicAdd(&sb[cur], acc);
                else atomicAdd(&a.bins[cur], acc);
            }
            cur = o;
            acc = 0.0;
        }
        acc = fma((double)v.re, (double)v.re, fma((double)v.im, (double)v.im, acc));
    }
    if (cur != 0xffffffffu) {
        if constexpr (SMEM) atomicAdd(&sb[cur], acc);
        else atomicAdd(&a.bins[cur], acc);
    }
    if constexpr (SMEM) {
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += blockDim.x)
            if (sb[i] != 0.0) atomicAdd(&a.bins[i], sb[i]);
    }
}

template <typename R>
__global__ void bins_to_out_kernel(const double* bins, uint64_t nb, void* out) {
    R* o = reinterpret_cast<R*>(out);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nb;
         i += (uint64_t)gridDim.x * blockDim.x)
        o[i] = (R)bins[i];
}


// ------------------------------------------------------------ readout / exchange helpers
// Full probabilities of one shard written at canonical positions: the
// amplitude at physical index (shard << nl | i) goes to out[o], o = sum over
// physical bits b of bit_b << cpos[b] (cpos = canonical bit of the logical
// qubit living at physical bit b).
struct ScatterArgs {
    uint64_t namp;
    uint64_t shard_bits;  // (shard index) << nl
    int nbits;            // total n
    int cpos[64];
    const void* psi;
    void* out;
};
template <typename R>
__global__ void __launch_bounds__(kThreads) prob_scatter_kernel(const __grid_constant__ ScatterArgs a) {
    const Cx<R>* psi = reinterpret_cast<const Cx<R>*>(a.psi);
    R* o = reinterpret_cast<R*>(a.out);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.namp;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = a.shard_bits | i;
        uint64_t y = 0;
        for (int b = 0; b < a.nbits; ++b) y |= ((x >> b) & 1ull) << a.cpos[b];
        const Cx<R> v = psi[i];
        o[y] = v.re * v.re + v.im * v.im;
    }
}

// Exchange for a local<->global qubit swap between two shards (virtual ranks
// on one device): shard a's amplitudes with local bit L = 1 trade places with
// shard b's amplitudes with local bit L = 0 (a has global bit 0, b has 1).
// When L is the top local bit both halves are contiguous blocks.
template <typename R>
__global__ void __launch_bounds__(kThreads) exchange_kernel(void* pa, void* pb, uint64_t nhalf, int L) {
    Cx<R>* a = reinterpret_cast<Cx<R>*>(pa);
    Cx<R>* b = reinterpret_cast<Cx<R>*>(pb);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nhalf;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = insert_zero(i, L);
        const uint64_t ia = lo | (1ull << L);
        const Cx<R> x = a[ia], y = b[lo];
        a[ia] = y;
        b[lo] = x;
    }
}

// ======================================================================
// Host launchers
// ======================================================================
inline int num_sms() {
    static int sms = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return sms;
}

template <typename KernelT>
inline uint64_t max_resident_blocks(KernelT kernel, int threads, size_t smem) {
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, threads, smem) != cudaSuccess || nb < 1) nb = 1;
    return (uint64_t)nb * (uint64_t)num_sms();
}

inline unsigned grid_for(uint64_t work_threads, uint64_t cap) {
    uint64_t b = (work_threads + kThreads - 1) / kThreads;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (unsigned)b;
}

// Split the fixed positions of a pass into low (vector/lane) and outer parts.
struct FixSplit {
    uint32_t low_mask = 0, low_val = 0;
    uint64_t fix_val = 0;
    int nout = 0;
    int out_pos[64];
};
inline FixSplit split_fixed(const Pass& p, int lb) {
    FixSplit f;
    for (int i = 0; i < p.nfix; ++i) {
        if (p.fpos[i] < lb) {
            f.low_mask |= 1u << p.fpos[i];
            if (p.fval[i]) f.low_val |= 1u << p.fpos[i];
        } else {
            f.out_pos[f.nout++] = p.fpos[i];
            if (p.fval[i]) f.fix_val |= 1ull << p.fpos[i];
        }
    }
    return f;
}

template <typename R>
inline Cx<R> to_cx(cd z) { return Cx<R>{(R)z.real(), (R)z.imag()}; }

// ---- simple path ----------------------------------------------------------
template <typename R, int K>
cudaError_t launch_simple_k(const Pass& p, const std::vector<cd>& dense, uint32_t touch, void* psi, int nl,
                            cudaStream_t st, LaunchStats& ls) {
    SimpleArgs<R, K> a;
    std::memset(&a, 0, sizeof(a));
    int all[64];
    int na = 0;
    for (int i = 0; i < K; ++i) all[na++] = p.tpos[i];
    for (int i = 0; i < p.nfix; ++i) {
        all[na++] = p.fpos[i];
        if (p.fval[i]) a.g.fix_val |= 1ull << p.fpos[i];
    }
    std::sort(all, all + na);
    a.g.nins = na;
    for (int i = 0; i < na; ++i) a.g.ins_pos[i] = all[i];
    for (int i = 0; i < K; ++i) a.g.tpos[i] = p.tpos[i];
    a.g.groups = 1ull << (nl - na);
    a.g.touch = touch;
    a.psi = psi;
    constexpr int D = 1 << K;
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c) a.m[r][c] = to_cx<R>(dense[(size_t)r * D + c]);
    static const uint64_t cap = max_resident_blocks(gate_simple_kernel<R, K>, kThreads, 0);
    gate_simple_kernel<R, K><<<grid_for(a.g.groups, cap), kThreads, 0, st>>>(a);
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t launch_simple(const Pass& p, void* psi, int nl, cudaStream_t st, LaunchStats& ls) {
    // every pass kind expressed as a small dense matrix on its targets
    int K = (p.kind == PK_PHASE || p.kind == PK_NEG) ? 0 : p.k;
    const int D = 1 << K;
    std::vector<cd> m((size_t)D * D, cd(0, 0));
    uint32_t touch = 0xffffffffu;
    switch (p.kind) {
        case PK_DENSE: m = p.m; touch = p.touch; break;
        case PK_X: m[1] = m[2] = 1; break;
        case PK_SWAP: m[0] = m[6] = m[9] = m[15] = 1; touch = 0x6; break;
        case PK_DIAG: for (int i = 0; i < D; ++i) m[(size_t)i * D + i] = p.m[i]; break;
        case PK_PHASE: m[0] = p.m[0]; break;
        case PK_NEG: m[0] = -1.0; break;
    }
    switch (K) {
        case 0: return launch_simple_k<R, 0>(p, m, touch, psi, nl, st, ls);
        case 1: return launch_simple_k<R, 1>(p, m, touch, psi, nl, st, ls);
        case 2: return launch_simple_k<R, 2>(p, m, touch, psi, nl, st, ls);
        case 3: return launch_simple_k<R, 3>(p, m, touch, psi, nl, st, ls);
        case 4: return launch_simple_k<R, 4>(p, m, touch, psi, nl, st, ls);
        case 5: return launch_simple_k<R, 5>(p, m, touch, psi, nl, st, ls);
    }
    return cudaErrorInvalidValue;
}

// ---- big-k path -------------------------------------------------------------
template <typename R>
cudaError_t launch_bigk(const Pass& p, void* psi, int nl, cudaStream_t st, void* scratch, size_t scratch_bytes,
                        LaunchStats& ls) {
    const int K = p.k, D = 1 << K;
    if (scratch == nullptr || scratch_bytes < sizeof(Cx<R>) * (size_t)D * D) return cudaErrorMemoryAllocation;
    std::vector<Cx<R>> h((size_t)D * D);
    for (size_t i = 0; i < h.size(); ++i) h[i] = to_cx<R>(p.m[i]);
    cudaError_t e = cudaMemcpyAsync(scratch, h.data(), h.size() * sizeof(Cx<R>), cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return e;
    BigKArgs a;
    std::memset(&a, 0, sizeof(a));
    int all[64];
    int na = 0;
    for (int i = 0; i < K; ++i) all[na++] = p.tpos[i];
    for (int i = 0; i < p.nfix; ++i) {
        all[na++] = p.fpos[i];
        if (p.fval[i]) a.fix_val |= 1ull << p.fpos[i];
    }
    std::sort(all, all + na);
    a.nins = na;
    for (int i = 0; i < na; ++i) a.ins_pos[i] = all[i];
    for (int i = 0; i < K; ++i) a.tpos[i] = p.tpos[i];
    a.k = K;
    a.groups = 1ull << (nl - na);
    a.psi = psi;
    a.m = scratch;
    uint64_t blocks = std::min<uint64_t>(a.groups, (uint64_t)num_sms() * 8);
    gate_bigk_kernel<R><<<(unsigned)blocks, D, 0, st>>>(a);
    ls.launches++;
    return cudaGetLastError();
}

// ---- warp path (dense / X / SWAP) ------------------------------------------
template <typename R, int K, int H, int KV, int MODE>
cudaError_t launch_warp(const WarpGeom& g, const std::vector<cd>& mcan, void* psi, cudaStream_t st,
                        LaunchStats& ls) {
    using Args = WarpArgs<R, K>;
    static Args* a = new Args;  // large parameter block; reused (launch copies it)
    std::memset(&a->g, 0, sizeof(a->g));
    a->g = g;
    a->psi = psi;
    constexpr int D = 1 << K;
    if (MODE == 0)
        for (int r = 0; r < D; ++r)
            for (int c = 0; c < D; ++c) a->m[r][c] = to_cx<R>(mcan[(size_t)r * D + c]);
    constexpr int V = VecT<R>::V;
    constexpr int U = (H + V >= 2) ? 1 : (1 << (2 - H - V));
    static const uint64_t cap = max_resident_blocks(gate_warp_kernel<R, K, H, KV, MODE>, kThreads, 0);
    const uint64_t threads = ((g.units + U - 1) / U) * 32;
    gate_warp_kernel<R, K, H, KV, MODE><<<grid_for(threads, cap), kThreads, 0, st>>>(*a);
    ls.launches++;
    return cudaGetLastError();
}

template <typename R, int K, int MODE, int H = 0>
cudaError_t dispatch_warp(int h, int kv, const WarpGeom& g, const std::vector<cd>& mcan, void* psi,
                          cudaStream_t st, LaunchStats& ls) {
    if constexpr (H > K) {
        return cudaErrorInvalidValue;
    } else {
        if (h == H) {
            if (kv == 0) return launch_warp<R, K, H, 0, MODE>(g, mcan, psi, st, ls);
            if constexpr (VecT<R>::V == 1 && K - H - 1 >= 0) return launch_warp<R, K, H, 1, MODE>(g, mcan, psi, st, ls);
            return cudaErrorInvalidValue;
        }
        return dispatch_warp<R, K, MODE, H + 1>(h, kv, g, mcan, psi, st, ls);
    }
}

template <typename R>
cudaError_t launch_gate(const Pass& p, void* psi, int nl, cudaStream_t st, LaunchStats& ls) {
    constexpr int V = VecT<R>::V;
    constexpr int LB = V + 5;
    const int K = p.k;
    // classify targets -> canonical order [outer | vector | lane]
    int canon[QJ_MAX_TARGETS];
    int nc = 0, H = 0, KV = 0, KL = 0;
    WarpGeom g;
    std::memset(&g, 0, sizeof(g));
    for (int i = 0; i < K; ++i)
        if (p.tpos[i] >= LB) { g.h_pos[H++] = p.tpos[i]; canon[nc++] = i; }
    for (int i = 0; i < K; ++i)
        if (V == 1 && p.tpos[i] == 0) { KV = 1; canon[nc++] = i; }
    for (int i = 0; i < K; ++i)
        if (p.tpos[i] < LB && !(V == 1 && p.tpos[i] == 0)) { g.l_pos[KL++] = p.tpos[i]; canon[nc++] = i; }
    FixSplit f = split_fixed(p, LB);
    const int nins = H + f.nout;
    if (nl - LB - nins < 0) return launch_simple<R>(p, psi, nl, st, ls);
    int ins[64];
    int ni = 0;
    for (int i = 0; i < H; ++i) ins[ni++] = g.h_pos[i];
    for (int i = 0; i < f.nout; ++i) ins[ni++] = f.out_pos[i];
    std::sort(ins, ins + ni);
    g.nins = ni;
    for (int i = 0; i < ni; ++i) g.ins_pos[i] = ins[i];
    g.fix_val = f.fix_val;
    g.low_mask = f.low_mask;
    g.low_val = f.low_val;
    g.units = 1ull << (nl - LB - nins);
    // sigma: canonical member index -> listed member index
    const int D = 1 << K;
    std::vector<int> sigma(D);
    for (int c = 0; c < D; ++c) {
        int s = 0;
        for (int j = 0; j < K; ++j)
            if ((c >> (K - 1 - j)) & 1) s |= 1 << (K - 1 - canon[j]);
        sigma[c] = s;
    }
    const uint32_t touch = (p.kind == PK_SWAP) ? 0x6u : (p.kind == PK_X ? 0x3u : p.touch);
    g.touch = 0;
    for (int c = 0; c < D; ++c)
        if ((touch >> sigma[c]) & 1u) g.touch |= 1u << c;
    std::vector<cd> mcan;
    if (p.kind == PK_DENSE) {
        mcan.resize((size_t)D * D);
        for (int r = 0; r < D; ++r)
            for (int c = 0; c < D; ++c) mcan[(size_t)r * D + c] = p.m[(size_t)sigma[r] * D + sigma[c]];
    }
    switch (p.kind) {
        case PK_X: return dispatch_warp<R, 1, 1>(H, KV, g, mcan, psi, st, ls);
        case PK_SWAP: return dispatch_warp<R, 2, 2>(H, KV, g, mcan, psi, st, ls);
        default: break;
    }
    switch (K) {
        case 1: return dispatch_warp<R, 1, 0>(H, KV, g, mcan, psi, st, ls);
        case 2: return dispatch_warp<R, 2, 0>(H, KV, g, mcan, psi, st, ls);
        case 3: return dispatch_warp<R, 3, 0>(H, KV, g, mcan, psi, st, ls);
        case 4: return dispatch_warp<R, 4, 0>(H, KV, g, mcan, psi, st, ls);
        case 5: return dispatch_warp<R, 5, 0>(H, KV, g, mcan, psi, st, ls);
    }
    return cudaErrorInvalidValue;
}

// ---- diagonal path ----------------------------------------------------------
template <typename R>
cudaError_t launch_diag(const Pass& p, void* psi, int nl, cudaStream_t st, LaunchStats& ls) {
    constexpr int V = VecT<R>::V;
    constexpr int LB = V + 5;
    FixSplit f = split_fixed(p, LB);
    if (nl - LB - f.nout < 0) return launch_simple<R>(p, psi, nl, st, ls);
    static DiagArgs<R>* a = new DiagArgs<R>;
    std::memset(a, 0, sizeof(*a));
    std::sort(f.out_pos, f.out_pos + f.nout);
    a->nins = f.nout;
    for (int i = 0; i < f.nout; ++i) a->ins_pos[i] = f.out_pos[i];
    a->fix_val = f.fix_val;
    a->low_mask = f.low_mask;
    a->low_val = f.low_val;
    a->units = 1ull << (nl - LB - f.nout);
    a->psi = psi;
    const uint64_t threads = ((a->units + 3) / 4) * 32;
    if (p.kind == PK_DIAG) {
        a->nt = p.k;
        for (int i = 0; i < p.k; ++i) a->tpos[i] = p.tpos[i];
        for (int i = 0; i < (1 << p.k); ++i) a->table[i] = to_cx<R>(p.m[i]);
        static const uint64_t cap = max_resident_blocks(diag_kernel<R, 0>, kThreads, 0);
        diag_kernel<R, 0><<<grid_for(threads, cap), kThreads, 0, st>>>(*a);
    } else if (p.kind == PK_PHASE) {
        a->phase = to_cx<R>(p.m[0]);
        static const uint64_t cap = max_resident_blocks(diag_kernel<R, 1>, kThreads, 0);
        diag_kernel<R, 1><<<grid_for(threads, cap), kThreads, 0, st>>>(*a);
    } else {
        static const uint64_t cap = max_resident_blocks(diag_kernel<R, 2>, kThreads, 0);
        diag_kernel<R, 2><<<grid_for(threads, cap), kThreads, 0, st>>>(*a);
    }
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_pass(const Pass& p, void* psi, int nl, cudaStream_t st, void* scratch, size_t scratch_bytes,
                     LaunchStats& ls) {
    switch (p.kind) {
        case PK_DIAG:
        case PK_PHASE:
        case PK_NEG:
            return launch_diag<R>(p, psi, nl, st, ls);
        default:
            if (p.k > 5) return launch_bigk<R>(p, psi, nl, st, scratch, scratch_bytes, ls);
            if constexpr (sizeof(R) == 4) {  // complex64 5-qubit blocks: tensor cores (dense_tc.cu)
                if (dense_tc_enabled() && dense_tc_supports(p, nl)) return run_dense_tc(p, psi, nl, st, ls);
            }
            return launch_gate<R>(p, psi, nl, st, ls);
    }
}

template <typename R>
cudaError_t run_init(void* psi, int nl, uint64_t basis_local, bool set_one, cudaStream_t st, LaunchStats& ls) {
    constexpr int V = VecT<R>::V;
    if (nl < V + 1) {
        init_scalar_kernel<R><<<1, 32, 0, st>>>(psi, 1ull << nl, basis_local, set_one ? 1 : 0);
    } else {
        const uint64_t nvec = 1ull << (nl - V);
        static const uint64_t cap = max_resident_blocks(init_kernel<R>, kThreads, 0);
        init_kernel<R><<<grid_for(nvec, cap), kThreads, 0, st>>>(psi, nvec, basis_local, set_one ? 1 : 0);
    }
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_prob_full(const void* psi, int nl, void* out, cudaStream_t st, LaunchStats& ls) {
    static const uint64_t cap = max_resident_blocks(prob_full_kernel<R>, kThreads, 0);
    prob_full_kernel<R><<<grid_for(1ull << nl, cap), kThreads, 0, st>>>(psi, out, 1ull << nl);
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_prob_marginal(const void* psi, int nl, const int* pos, const int* gval, int nq, double* bins,
                              cudaStream_t st, LaunchStats& ls) {
    MargArgs a;
    std::memset(&a, 0, sizeof(a));
    a.namp = 1ull << nl;
    a.nq = nq;
    for (int i = 0; i < nq; ++i) {
        a.pos[i] = pos[i];
        a.cbit[i] = gval ? gval[i] : 0;
    }
    a.bins = bins;
    a.psi = psi;
    int minpos = 64;
    for (int i = 0; i < nq; ++i)
        if (pos[i] >= 0) minpos = std::min(minpos, pos[i]);
    const int cb = std::min(nl, 16);
    if (minpos >= cb && cb >= VecT<R>::V + 8) {
        prob_chunk_kernel<R><<<(unsigned)(1ull << (nl - cb)), kThreads, 0, st>>>(a, cb);
    } else {
        // grid = a power of two so the stride is a multiple of 2^(max listed bit + 1)
        // whenever that fits (then every thread's bin is fixed)
        const int nbytes = (nl + 7) / 8;
        const bool smem = nq <= 12;
        const uint64_t cap = smem ? max_resident_blocks(prob_marg_kernel<R, true>, kThreads, 0)
                                  : max_resident_blocks(prob_marg_kernel<R, false>, kThreads, 0);
        uint64_t g = 1;
        while (g * 2 <= cap && g * 2 * kThreads <= a.namp) g *= 2;
        if (smem) prob_marg_kernel<R, true><<<(unsigned)g, kThreads, 0, st>>>(a, nbytes);
        else prob_marg_kernel<R, false><<<(unsigned)g, kThreads, 0, st>>>(a, nbytes);
    }
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_bins_to_out(const double* bins, uint64_t nbins, void* out, cudaStream_t st, LaunchStats& ls) {
    bins_to_out_kernel<R><<<grid_for(nbins, 1184), kThreads, 0, st>>>(bins, nbins, out);
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_prob_scatter(const void* psi, int nl, uint64_t shard, int n, const int* cpos, void* out,
                             cudaStream_t st, LaunchStats& ls) {
    ScatterArgs a;
    std::memset(&a, 0, sizeof(a));
    a.namp = 1ull << nl;
    a.shard_bits = shard << nl;
    a.nbits = n;
    for (int b = 0; b < n; ++b) a.cpos[b] = cpos[b];
    a.psi = psi;
    a.out = out;
    static const uint64_t cap = max_resident_blocks(prob_scatter_kernel<R>, kThreads, 0);
    prob_scatter_kernel<R><<<grid_for(a.namp, cap), kThreads, 0, st>>>(a);
    ls.launches++;
    return cudaGetLastError();
}

template <typename R>
cudaError_t run_exchange(void* a, void* b, int nl, int L, cudaStream_t st, LaunchStats& ls) {
    const uint64_t nhalf = 1ull << (nl - 1);
    static const uint64_t cap = max_resident_blocks(exchange_kernel<R>, kThreads, 0);
    exchange_kernel<R><<<grid_for(nhalf, cap), kThreads, 0, st>>>(a, b, nhalf, L);
    ls.launches++;
    return cudaGetLastError();
}

#define QJ_INSTANTIATE(R)                                                                                    \
    template cudaError_t run_pass<R>(const Pass&, void*, int, cudaStream_t, void*, size_t, LaunchStats&);    \
    template cudaError_t run_init<R>(void*, int, uint64_t, bool, cudaStream_t, LaunchStats&);                \
    template cudaError_t run_prob_full<R>(const void*, int, void*, cudaStream_t, LaunchStats&);              \
    template cudaError_t run_prob_marginal<R>(const void*, int, const int*, const int*, int, double*,        \
                                              cudaStream_t, LaunchStats&);                                   \
    template cudaError_t run_bins_to_out<R>(const double*, uint64_t, void*, cudaStream_t, LaunchStats&);   \
    template cudaError_t run_prob_scatter<R>(const void*, int, uint64_t, int, const int*, void*, cudaStream_t, \
                                             LaunchStats&);                                                  \
    template cudaError_t run_exchange<R>(void*, void*, int, int, cudaStream_t, LaunchStats&);

}  // namespace qj
