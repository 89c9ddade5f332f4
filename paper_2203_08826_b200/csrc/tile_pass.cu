// tile_pass.cu -- the fused window tile pass kernel (see tile.h) and its
// launcher, which lowers a host TileSpec into the kernel's parameter block
// plus a device program buffer (terms, slots, matrices, anchored factors).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>

#include "tile.h"

namespace qj {

// XOR swizzle of the tile-local amplitude index into a shared-memory slot.
// Linear over GF(2) (slot(a ^ b) = slot(a) ^ slot(b)), so per-register offsets
// can be swizzled independently of the per-thread base.  A quarter warp of
// 16-byte (c128) / half warp of 8-byte (c64) accesses is conflict free when
// its lane bits map to window bits of distinct residues mod 3 (mod 4).
template <typename R>
__host__ __device__ __forceinline__ uint32_t swz(uint32_t i);
template <>
__host__ __device__ __forceinline__ uint32_t swz<double>(uint32_t i) {
    return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9)) & 7u);
}
template <>
__host__ __device__ __forceinline__ uint32_t swz<float>(uint32_t i) {
    return i ^ (((i >> 4) ^ (i >> 8)) & 15u);
}

template <typename R>
__device__ __forceinline__ Cx<R> cone() {
    return Cx<R>{R(1), R(0)};
}

// ---------------------------------------------------------------- gate ops on registers
template <typename R, int A, bool C>
__device__ __forceinline__ void op_h(Cx<R> (&v)[TILE_NREG], R s, uint32_t crm, uint32_t crv, bool ok) {
#pragma unroll
    for (int j = 0; j < TILE_NREG / 2; ++j) {
        const int lo = ((j >> A) << (A + 1)) | (j & ((1 << A) - 1));
        const int hi = lo | (1 << A);
        if (!C || (ok && ((uint32_t)lo & crm) == crv)) {
            const Cx<R> x = v[lo], y = v[hi];
            v[lo] = Cx<R>{(x.re + y.re) * s, (x.im + y.im) * s};
            v[hi] = Cx<R>{(x.re - y.re) * s, (x.im - y.im) * s};
        }
    }
}

template <typename R, int A, bool C>
__device__ __forceinline__ void op_u1(Cx<R> (&v)[TILE_NREG], const Cx<R>* m, uint32_t crm, uint32_t crv, bool ok) {
    const Cx<R> m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
#pragma unroll
    for (int j = 0; j < TILE_NREG / 2; ++j) {
        const int lo = ((j >> A) << (A + 1)) | (j & ((1 << A) - 1));
        const int hi = lo | (1 << A);
        if (!C || (ok && ((uint32_t)lo & crm) == crv)) {
            const Cx<R> x = v[lo], y = v[hi];
            Cx<R> o0{R(0), R(0)}, o1{R(0), R(0)};
            cfma(o0, m00, x);
            cfma(o0, m01, y);
            cfma(o1, m10, x);
            cfma(o1, m11, y);
            v[lo] = o0;
            v[hi] = o1;
        }
    }
}

template <typename R, int A, bool C>
__device__ __forceinline__ void op_x(Cx<R> (&v)[TILE_NREG], uint32_t crm, uint32_t crv, bool ok) {
#pragma unroll
    for (int j = 0; j < TILE_NREG / 2; ++j) {
        const int lo = ((j >> A) << (A + 1)) | (j & ((1 << A) - 1));
        const int hi = lo | (1 << A);
        if (!C || (ok && ((uint32_t)lo & crm) == crv)) {
            const Cx<R> x = v[lo];
            v[lo] = v[hi];
            v[hi] = x;
        }
    }
}

// 4x4 on register bits A (matrix MSB) and B
template <typename R, int A, int B, bool C>
__device__ __forceinline__ void op_u2(Cx<R> (&v)[TILE_NREG], const Cx<R>* m, uint32_t crm, uint32_t crv, bool ok) {
    constexpr int LO = A < B ? A : B, HI = A < B ? B : A;
#pragma unroll
    for (int j = 0; j < TILE_NREG / 4; ++j) {
        int base = ((j >> LO) << (LO + 1)) | (j & ((1 << LO) - 1));
        base = ((base >> HI) << (HI + 1)) | (base & ((1 << HI) - 1));
        if (C && !(ok && ((uint32_t)base & crm) == crv)) continue;
        int id[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) id[q] = base | (((q >> 1) & 1) << A) | ((q & 1) << B);
        Cx<R> in[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) in[q] = v[id[q]];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            Cx<R> o{R(0), R(0)};
#pragma unroll
            for (int c = 0; c < 4; ++c) cfma(o, m[r * 4 + c], in[c]);
            v[id[r]] = o;
        }
    }
}

template <typename R, int A, int B, bool C>
__device__ __forceinline__ void op_swap(Cx<R> (&v)[TILE_NREG], uint32_t crm, uint32_t crv, bool ok) {
#pragma unroll
    for (int j = 0; j < TILE_NREG; ++j) {
        if (((j >> A) & 1) == 1 && ((j >> B) & 1) == 0) {
            const int k = j ^ (1 << A) ^ (1 << B);
            if (!C || (ok && ((uint32_t)j & crm) == crv)) {
                const Cx<R> x = v[j];
                v[j] = v[k];
                v[k] = x;
            }
        }
    }
}

// ---------------------------------------------------------------- phase runs
// Multiply the registers whose bit J equals X (J < 0: all) by g.  All register
// selection is compile-time: no predicated multiplies are issued.
template <typename R, int ANC, int VAL, int J, int X>
__device__ __forceinline__ void mul_sel(Cx<R> (&v)[TILE_NREG], Cx<R> g) {
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) {
        if (ANC >= 0 && ((r >> ANC) & 1) != VAL) continue;
        if (J >= 0 && ((r >> J) & 1) != X) continue;
        v[r] = cmul(g, v[r]);
    }
}

// Per register bit J: multiply by g1 where x_J = 1 and by g0 where x_J = 0
// (skipped when only1).  ANC/VAL restrict to registers with anchor bit = VAL.
template <typename R, int ANC, int VAL, int J>
__device__ __forceinline__ void mul_pair(Cx<R> (&v)[TILE_NREG], Cx<R> g0, Cx<R> g1, bool only1) {
    mul_sel<R, ANC, VAL, J, 1>(v, g1);
    if (!only1) mul_sel<R, ANC, VAL, J, 0>(v, g0);
}

template <typename R, int ANC, int VAL>
__device__ __forceinline__ void mul_pairs(Cx<R> (&v)[TILE_NREG], const Cx<R> (&g)[TILE_R][2], uint32_t use,
                                          uint32_t only1) {
    if (((use >> 0) & 1) && ANC != 0) mul_pair<R, ANC, VAL, 0>(v, g[0][0], g[0][1], (only1 >> 0) & 1);
    if (((use >> 1) & 1) && ANC != 1) mul_pair<R, ANC, VAL, 1>(v, g[1][0], g[1][1], (only1 >> 1) & 1);
    if (((use >> 2) & 1) && ANC != 2) mul_pair<R, ANC, VAL, 2>(v, g[2][0], g[2][1], (only1 >> 2) & 1);
    if (((use >> 3) & 1) && ANC != 3) mul_pair<R, ANC, VAL, 3>(v, g[3][0], g[3][1], (only1 >> 3) & 1);
}

// SLOT run: scalar (S, CT slots, per-thread table TA, generic scalar terms),
// per-register-bit pairs (CR slots, per-thread table TB, generic single-R
// terms) and a uniform register-pattern table PT.
template <typename R>
__device__ __forceinline__ void apply_slot_run(const TileArgs<R>& a, const TRunDesc& d, Cx<R> (&v)[TILE_NREG],
                                               uint64_t tfull, int tid, const Cx<R>* tab) {
    const TTerm<R>* terms = reinterpret_cast<const TTerm<R>*>(a.tables + a.lay.terms);
    const Cx<R>* fac = reinterpret_cast<const Cx<R>*>(a.tables + a.lay.fac);
    Cx<R> sc = cone<R>();
    if (d.has_scalar) {
        if (d.s_slot >= 0) sc = tab[d.s_slot];
        for (int i = 0; i < TILE_T; ++i) {
            const int sl = d.ct_slot[i][(tid >> i) & 1];
            if (sl >= 0) sc = cmul(sc, tab[sl]);
        }
        if (d.ta >= 0) sc = cmul(sc, fac[d.ta + tid]);
    }
    Cx<R> pr[TILE_R][2];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int sl = d.cr_slot[j][b];
            pr[j][b] = sl >= 0 ? tab[sl] : cone<R>();
            if (d.tb >= 0) pr[j][b] = cmul(pr[j][b], fac[d.tb + (tid * TILE_R + j) * 2 + b]);
        }
    for (int t = d.l0; t < d.l1; ++t) {
        const TTerm<R> T = terms[t];
        if ((tfull & T.cmask) != T.cval) continue;
        const uint32_t rm = T.rmask;
        if (rm == 0) {
            sc = cmul(sc, T.f);
        } else if ((rm & (rm - 1)) == 0) {
#pragma unroll
            for (int j = 0; j < TILE_R; ++j)
                if (rm == (1u << j)) {
                    if (T.rval & (1u << j)) pr[j][1] = cmul(pr[j][1], T.f);
                    else pr[j][0] = cmul(pr[j][0], T.f);
                }
        } else {
#pragma unroll
            for (int r = 0; r < TILE_NREG; ++r)
                if (((uint32_t)r & rm) == T.rval) v[r] = cmul(T.f, v[r]);
        }
    }
    if (d.has_scalar) mul_sel<R, -1, 0, -1, 0>(v, sc);
    mul_pairs<R, -1, 0>(v, pr, d.ru, d.r0one);
    if (d.pt >= 0) {
#pragma unroll
        for (int r = 0; r < TILE_NREG; ++r) v[r] = cmul(fac[d.pt + r], v[r]);
    }
}

// ANCHORED run on register bit ANC, value VAL: amplitudes with x_ANC = VAL get
// slot(tile) * prod_{thread bits} g_T[x] * prod_{other register bits} g_R[x].
template <typename R, int ANC, int VAL>
__device__ __forceinline__ void anchor_apply(const TRunDesc& d, const Cx<R>* f, const Cx<R>* fbase,
                                             Cx<R> (&v)[TILE_NREG], int tid, const Cx<R>* tab) {
    Cx<R> F = d.aslot[VAL] >= 0 ? tab[d.aslot[VAL]] : cone<R>();
    if (d.ft >= 0) F = cmul(F, reinterpret_cast<const Cx<R>*>(fbase)[d.ft + VAL * TILE_THREADS + tid]);
    const uint32_t rm = d.rm[VAL] & ~(1u << ANC), r1 = d.r1only[VAL];
    Cx<R> g[TILE_R][2];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j) {
        g[j][0] = f[2 * TILE_T * 2 + (VAL * TILE_R + j) * 2];
        g[j][1] = f[2 * TILE_T * 2 + (VAL * TILE_R + j) * 2 + 1];
    }
    // fold F into one partner bit's factor pair (saves a sweep over the anchor registers)
    uint32_t only1 = r1;
    if (rm) {
        const uint32_t both = rm & ~r1;
        const int j0 = __ffs(both ? both : rm) - 1;
#pragma unroll
        for (int j = 0; j < TILE_R; ++j)
            if (j == j0) {
                g[j][0] = ((r1 >> j) & 1) ? F : cmul(F, g[j][0]);
                g[j][1] = cmul(F, g[j][1]);
            }
        only1 &= ~(1u << j0);
    } else {
        mul_sel<R, ANC, VAL, -1, 0>(v, F);
    }
    mul_pairs<R, ANC, VAL>(v, g, rm, only1);
}

template <typename R, int ANC>
__device__ __forceinline__ void anchor_run(const TileArgs<R>& a, const TRunDesc& d, Cx<R> (&v)[TILE_NREG], int tid,
                                           const Cx<R>* tab) {
    const Cx<R>* fb = reinterpret_cast<const Cx<R>*>(a.tables + a.lay.fac);
    const Cx<R>* f = fb + d.fac;
    if (d.vmask & 1) anchor_apply<R, ANC, 0>(d, f, fb, v, tid, tab);
    if (d.vmask & 2) anchor_apply<R, ANC, 1>(d, f, fb, v, tid, tab);
}

template <typename R, bool C>
__device__ __forceinline__ void apply_op_t(const TileArgs<R>& a, const TOp& op, Cx<R> (&v)[TILE_NREG], uint64_t tfull,
                                         int tid, const Cx<R>* tab) {
    const bool ok = op.cx < 0 || (tfull & a.cx[op.cx][0]) == a.cx[op.cx][1];
    const uint32_t crm = op.cr_mask, crv = op.cr_val;
    const Cx<R>* mats = reinterpret_cast<const Cx<R>*>(a.tables + a.lay.mats);
    switch (op.type) {
        case TO_H: {
            const R hs = mats[op.idx].re;  // the caller's own 1/sqrt(2)
            switch (op.a) {
                case 0: op_h<R, 0, false>(v, hs, crm, crv, ok); break;
                case 1: op_h<R, 1, false>(v, hs, crm, crv, ok); break;
                case 2: op_h<R, 2, false>(v, hs, crm, crv, ok); break;
                default: op_h<R, 3, false>(v, hs, crm, crv, ok); break;
            }
            break;
        }
        case TO_U1: {
            const Cx<R>* m = mats + op.idx;
            switch (op.a) {
                case 0: op_u1<R, 0, C>(v, m, crm, crv, ok); break;
                case 1: op_u1<R, 1, C>(v, m, crm, crv, ok); break;
                case 2: op_u1<R, 2, C>(v, m, crm, crv, ok); break;
                default: op_u1<R, 3, C>(v, m, crm, crv, ok); break;
            }
            break;
        }
        case TO_X:
            switch (op.a) {
                case 0: op_x<R, 0, C>(v, crm, crv, ok); break;
                case 1: op_x<R, 1, C>(v, crm, crv, ok); break;
                case 2: op_x<R, 2, C>(v, crm, crv, ok); break;
                default: op_x<R, 3, C>(v, crm, crv, ok); break;
            }
            break;
        case TO_U2: {
            const Cx<R>* m = mats + op.idx;
            switch (op.a * 4 + op.b) {
                case 1: op_u2<R, 0, 1, C>(v, m, crm, crv, ok); break;
                case 2: op_u2<R, 0, 2, C>(v, m, crm, crv, ok); break;
                case 3: op_u2<R, 0, 3, C>(v, m, crm, crv, ok); break;
                case 4: op_u2<R, 1, 0, C>(v, m, crm, crv, ok); break;
                case 6: op_u2<R, 1, 2, C>(v, m, crm, crv, ok); break;
                case 7: op_u2<R, 1, 3, C>(v, m, crm, crv, ok); break;
                case 8: op_u2<R, 2, 0, C>(v, m, crm, crv, ok); break;
                case 9: op_u2<R, 2, 1, C>(v, m, crm, crv, ok); break;
                case 11: op_u2<R, 2, 3, C>(v, m, crm, crv, ok); break;
                case 12: op_u2<R, 3, 0, C>(v, m, crm, crv, ok); break;
                case 13: op_u2<R, 3, 1, C>(v, m, crm, crv, ok); break;
                default: op_u2<R, 3, 2, C>(v, m, crm, crv, ok); break;
            }
            break;
        }
        case TO_SWAP: {
            const int lo = op.a < op.b ? op.a : op.b, hi = op.a < op.b ? op.b : op.a;
            switch (lo * 4 + hi) {
                case 1: op_swap<R, 1, 0, C>(v, crm, crv, ok); break;
                case 2: op_swap<R, 2, 0, C>(v, crm, crv, ok); break;
                case 3: op_swap<R, 3, 0, C>(v, crm, crv, ok); break;
                case 6: op_swap<R, 2, 1, C>(v, crm, crv, ok); break;
                case 7: op_swap<R, 3, 1, C>(v, crm, crv, ok); break;
                default: op_swap<R, 3, 2, C>(v, crm, crv, ok); break;
            }
            break;
        }
        default: {
            const TRunDesc& d = a.runs[op.idx];
            if (d.kind == RUN_ANCHOR) {
                switch (d.anc) {
                    case 0: anchor_run<R, 0>(a, d, v, tid, tab); break;
                    case 1: anchor_run<R, 1>(a, d, v, tid, tab); break;
                    case 2: anchor_run<R, 2>(a, d, v, tid, tab); break;
                    default: anchor_run<R, 3>(a, d, v, tid, tab); break;
                }
            } else {
                apply_slot_run(a, d, v, tfull, tid, tab);
            }
            break;
        }
    }
}

template <typename R>
__device__ __forceinline__ void apply_op(const TileArgs<R>& a, const TOp& op, Cx<R> (&v)[TILE_NREG], uint64_t tfull,
                                         int tid, const Cx<R>* tab) {
    apply_op_t<R, true>(a, op, v, tfull, tid, tab);  // predicated form: the unpredicated one spills
}

// Physical / window-local offsets of a thread's index bits in segment s,
// from host-built nibble tables (thread bits 0-3 and 4-7).
template <typename R>
__device__ __forceinline__ uint64_t thread_phys(const TileArgs<R>& a, int s, int tid) {
    return a.tph[s][0][tid & 15] | a.tph[s][1][tid >> 4];
}
template <typename R>
__device__ __forceinline__ uint32_t thread_loc(const TileArgs<R>& a, int s, int tid) {
    return a.tlo[s][0][tid & 15] | a.tlo[s][1][tid >> 4];
}

template <typename R>
__global__ void __launch_bounds__(TILE_THREADS, 2) tile_kernel(const __grid_constant__ TileArgs<R> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Cx<R>* sm = reinterpret_cast<Cx<R>*>(smraw);
    Cx<R>* tab = sm + (1 << TILE_W);
    const int tid = threadIdx.x;
    Cx<R>* psi = reinterpret_cast<Cx<R>*>(a.psi);
    const TSlot* slots = reinterpret_cast<const TSlot*>(a.tables + a.lay.slots);
    const TTerm<R>* terms = reinterpret_cast<const TTerm<R>*>(a.tables + a.lay.terms);

    for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        uint64_t tb = tile;
#pragma unroll
        for (int i = 0; i < TILE_W; ++i) tb = insert_zero(tb, a.wpos[i]);
        // per-tile products of the tile-dependent phase terms
        for (int e = tid; e < a.nslots; e += TILE_THREADS) {
            Cx<R> p = cone<R>();
            const TSlot sl = slots[e];
            for (uint32_t t = sl.t0; t < sl.t1; ++t)
                if ((tb & terms[t].cmask) == terms[t].cval) p = cmul(p, terms[t].f);
            tab[e] = p;
        }
        Cx<R> v[TILE_NREG];
        {
            const TSeg& S = a.seg[0];
            const uint64_t base = tb | thread_phys(a, 0, tid);
            uint64_t rm[TILE_R];
#pragma unroll
            for (int j = 0; j < TILE_R; ++j) rm[j] = 1ull << a.wpos[S.rbits[j]];
#pragma unroll
            for (int r = 0; r < TILE_NREG; ++r) {
                uint64_t x = base;
#pragma unroll
                for (int j = 0; j < TILE_R; ++j)
                    if ((r >> j) & 1) x |= rm[j];
                v[r] = load_amp(psi, x);
            }
        }
        __syncthreads();  // tab ready
        for (int s = 0; s < a.nseg; ++s) {
            const TSeg& S = a.seg[s];
            if (s > 0) {
                const TSeg& P = a.seg[s - 1];
                const uint32_t bp = swz<R>(thread_loc(a, s - 1, tid));
                uint32_t sp[TILE_R];
#pragma unroll
                for (int j = 0; j < TILE_R; ++j) sp[j] = swz<R>(1u << P.rbits[j]);
                __syncthreads();
#pragma unroll
                for (int r = 0; r < TILE_NREG; ++r) {
                    uint32_t x = bp;
#pragma unroll
                    for (int j = 0; j < TILE_R; ++j)
                        if ((r >> j) & 1) x ^= sp[j];
                    sm[x] = v[r];
                }
                __syncthreads();
                const uint32_t bn = swz<R>(thread_loc(a, s, tid));
                uint32_t sn[TILE_R];
#pragma unroll
                for (int j = 0; j < TILE_R; ++j) sn[j] = swz<R>(1u << S.rbits[j]);
#pragma unroll
                for (int r = 0; r < TILE_NREG; ++r) {
                    uint32_t x = bn;
#pragma unroll
                    for (int j = 0; j < TILE_R; ++j)
                        if ((r >> j) & 1) x ^= sn[j];
                    v[r] = sm[x];
                }
            }
            const uint64_t tfull = tb | thread_phys(a, s, tid);
            for (int o = S.op0; o < S.op1; ++o) apply_op(a, a.ops[o], v, tfull, tid, tab);
        }
        {
            const TSeg& S = a.seg[a.nseg - 1];
            const uint64_t base = tb | thread_phys(a, a.nseg - 1, tid);
            uint64_t rm[TILE_R];
#pragma unroll
            for (int j = 0; j < TILE_R; ++j) rm[j] = 1ull << a.wpos[S.rbits[j]];
#pragma unroll
            for (int r = 0; r < TILE_NREG; ++r) {
                uint64_t x = base;
#pragma unroll
                for (int j = 0; j < TILE_R; ++j)
                    if ((r >> j) & 1) x |= rm[j];
                store_amp(a.psi, x, v[r]);
            }
        }
        __syncthreads();  // tab / smem reuse by the next tile
    }
}

// ======================================================================
// Staging ring
// ======================================================================
cudaError_t TileStaging::init() {
    if (host) return cudaSuccess;
    cudaError_t e = cudaMallocHost(&host, kSlots * kBytes);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&dev, kSlots * kBytes);
    if (e != cudaSuccess) return e;
    for (int i = 0; i < kSlots; ++i) {
        e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

void TileStaging::release() {
    for (int i = 0; i < kSlots; ++i)
        if (ev[i]) {
            cudaEventSynchronize(ev[i]);
            cudaEventDestroy(ev[i]);
            ev[i] = nullptr;
        }
    if (host) cudaFreeHost(host);
    if (dev) cudaFree(dev);
    host = dev = nullptr;
}

// ======================================================================
// Launcher: TileSpec (physical bits, host) -> TileArgs<R> + program buffer
// ======================================================================
namespace {

int popc64(uint64_t x) { return __builtin_popcountll(x); }

// H up to rounding of 1/sqrt(2): m00 = m01 = m10 = -m11 real; the kernel then
// uses m00 itself as the scale ((x +- y) * m00).
bool is_hadamard(const std::vector<cd>& m, double tol) {
    const double s = m[0].real();
    return m[0].imag() == 0 && m[1] == m[0] && m[2] == m[0] && m[3] == -m[0] &&
           std::fabs(s - 0.70710678118654752440) <= tol;
}

}  // namespace

// Lower a TileSpec into kernel parameters + program-buffer bytes (host only).
// Returns false when the pass exceeds a capacity (the planner then splits it).
template <typename R>
bool lower_tile(const TileSpec& t, int nl, TileArgs<R>* a, std::vector<unsigned char>& blob) {
    std::memset(a, 0, sizeof(TileArgs<R>));
    if ((int)t.segs.size() < 1 || (int)t.segs.size() > TILE_MAXSEG) return false;
    a->ntiles = 1ull << (nl - TILE_W);
    a->nseg = (int)t.segs.size();
    a->nops = (int)t.ops.size();
    uint64_t wmask = 0;
    for (int i = 0; i < TILE_W; ++i) {
        a->wpos[i] = t.wpos[i];
        wmask |= 1ull << t.wpos[i];
    }
    std::vector<TTerm<R>> terms;      // slot terms then L terms
    std::vector<TSlot> slots;
    std::vector<Cx<R>> mats, fac;
    std::vector<TTerm<R>> lterms_all; // appended after slot terms; ranges patched later
    struct LRange {
        int run;
        size_t b, e;
    };
    std::vector<LRange> lranges;
    int ncx = 0, nruns = 0;
    auto new_slot = [&](const std::vector<TTerm<R>>& ts) -> int {
        TSlot sl;
        sl.t0 = (uint32_t)terms.size();
        for (auto& x : ts) terms.push_back(x);
        sl.t1 = (uint32_t)terms.size();
        slots.push_back(sl);
        return (int)slots.size() - 1;
    };
    auto to_r = [](cd z) { return Cx<R>{(R)z.real(), (R)z.imag()}; };
    std::vector<TOp> ops;
    for (int si = 0; si < a->nseg; ++si) {
        const TSeg& S = t.segs[si];
        a->seg[si] = S;
        for (int half = 0; half < 2; ++half)
            for (int nib = 0; nib < 16; ++nib) {
                uint64_t ph = 0;
                uint32_t lo = 0;
                for (int q = 0; q < 4; ++q)
                    if ((nib >> q) & 1) {
                        const int wb = S.tbits[half * 4 + q];
                        ph |= 1ull << t.wpos[wb];
                        lo |= 1u << wb;
                    }
                a->tph[si][half][nib] = ph;
                a->tlo[si][half][nib] = lo;
            }
        a->seg[si].op0 = (uint16_t)ops.size();
        uint64_t rmask = 0;
        int rl_of_bit[64], tl_of_bit[64];
        for (int b = 0; b < 64; ++b) rl_of_bit[b] = tl_of_bit[b] = -1;
        for (int j = 0; j < TILE_R; ++j) {
            const int b = t.wpos[S.rbits[j]];
            rmask |= 1ull << b;
            rl_of_bit[b] = j;
        }
        for (int i = 0; i < TILE_T; ++i) tl_of_bit[t.wpos[S.tbits[i]]] = i;
        auto cls = [&](int b) { return !((wmask >> b) & 1) ? 'C' : (((rmask >> b) & 1) ? 'R' : 'T'); };
        for (int o = S.op0; o < S.op1; ++o) {
            const HOp& h = t.ops[o];
            TOp op;
            std::memset(&op, 0, sizeof(op));
            op.cx = -1;
            const uint64_t crp = h.cmask & rmask, cxp = h.cmask & ~rmask;
            for (int b = 0; b < 64; ++b)
                if ((crp >> b) & 1) op.cr_mask |= (uint8_t)(1u << rl_of_bit[b]);
            op.cr_val = op.cr_mask;
            if (cxp) {
                int found = -1;
                for (int c = 0; c < ncx; ++c)
                    if (a->cx[c][0] == cxp) found = c;
                if (found < 0) {
                    if (ncx >= TILE_MAXCX) return false;
                    a->cx[ncx][0] = cxp;
                    a->cx[ncx][1] = cxp;
                    found = ncx++;
                }
                op.cx = (int16_t)found;
            }
            if (h.type == TO_U1 || h.type == TO_X || h.type == TO_H) {
                const int j = rl_of_bit[h.t[0]];
                if (j < 0) return false;
                op.a = (uint8_t)j;
                if (h.type == TO_X) {
                    op.type = TO_X;
                } else if (h.cmask == 0 && is_hadamard(h.m, sizeof(R) == 8 ? 1e-15 : 1e-7)) {
                    op.type = TO_H;
                    op.idx = (uint16_t)mats.size();
                    mats.push_back(to_r(h.m[0]));
                } else {
                    op.type = TO_U1;
                    op.idx = (uint16_t)mats.size();
                    for (int q = 0; q < 4; ++q) mats.push_back(to_r(h.m[q]));
                }
                ops.push_back(op);
                continue;
            }
            if (h.type == TO_U2 || h.type == TO_SWAP) {
                const int j0 = rl_of_bit[h.t[0]], j1 = rl_of_bit[h.t[1]];
                if (j0 < 0 || j1 < 0 || j0 == j1) return false;
                op.type = (uint8_t)h.type;
                op.a = (uint8_t)j0;
                op.b = (uint8_t)j1;
                if (h.type == TO_U2) {
                    op.idx = (uint16_t)mats.size();
                    for (int q = 0; q < 16; ++q) mats.push_back(to_r(h.m[q]));
                }
                ops.push_back(op);
                continue;
            }
            if (h.type != TO_RUN) return false;
            // ---- phase run: one SLOT run (+ per-thread tables) and ANCHORED runs on register bits
            std::vector<const HTerm*> slotable, rest;
            for (const HTerm& ht : h.terms) {
                if (ht.f == cd(1, 0)) continue;
                int nw = 0;
                for (int b = 0; b < 64; ++b)
                    if (((ht.mask >> b) & 1) && cls(b) != 'C') ++nw;
                (nw <= 1 ? slotable : rest).push_back(&ht);
            }
            // anchored groups on register bits: terms of exactly two bits, one of them
            // the anchor; greedy by the register bit shared by most remaining terms
            std::vector<std::pair<int, std::vector<const HTerm*>>> groups;
            while (!rest.empty()) {
                std::map<int, int> cnt;
                for (auto* ht : rest) {
                    if (popc64(ht->mask) != 2) continue;
                    for (int b = 0; b < 64; ++b)
                        if (((ht->mask >> b) & 1) && cls(b) == 'R') cnt[b]++;
                }
                int best = -1, bc = 0;
                for (auto& kv : cnt)
                    if (kv.second > bc) {
                        bc = kv.second;
                        best = kv.first;
                    }
                if (best < 0) break;
                std::vector<const HTerm*> g, keep;
                for (auto* ht : rest) ((popc64(ht->mask) == 2 && ((ht->mask >> best) & 1)) ? g : keep).push_back(ht);
                groups.push_back({best, g});
                rest.swap(keep);
            }
            // the rest: window-only terms with <= 1 register bit (or register-only) go to
            // host-built per-thread tables; anything else is a generic L term
            std::vector<cd> TA, TB, PT;
            std::vector<const HTerm*> generic;
            for (auto* ht : rest) {
                const uint64_t cb = ht->mask & ~wmask, rb = ht->mask & rmask, tbm = ht->mask & wmask & ~rmask;
                const int nr = popc64(rb);
                if (cb || (nr >= 2 && tbm)) {
                    generic.push_back(ht);
                    continue;
                }
                if (nr >= 2) {  // register-only pattern: uniform table
                    if (PT.empty()) PT.assign(TILE_NREG, cd(1, 0));
                    for (int r = 0; r < TILE_NREG; ++r) {
                        bool m = true;
                        for (int b = 0; b < 64; ++b)
                            if ((rb >> b) & 1) m &= (((r >> rl_of_bit[b]) & 1) == (int)((ht->val >> b) & 1));
                        if (m) PT[r] *= ht->f;
                    }
                    continue;
                }
                for (int tid = 0; tid < TILE_THREADS; ++tid) {
                    bool m = true;
                    for (int b = 0; b < 64; ++b)
                        if ((tbm >> b) & 1) m &= (((tid >> tl_of_bit[b]) & 1) == (int)((ht->val >> b) & 1));
                    if (!m) continue;
                    if (nr == 0) {
                        if (TA.empty()) TA.assign(TILE_THREADS, cd(1, 0));
                        TA[tid] *= ht->f;
                    } else {
                        if (TB.empty()) TB.assign((size_t)TILE_THREADS * TILE_R * 2, cd(1, 0));
                        const int b = __builtin_ctzll(rb);
                        TB[((size_t)tid * TILE_R + rl_of_bit[b]) * 2 + ((ht->val >> b) & 1)] *= ht->f;
                    }
                }
            }
            if (!slotable.empty() || !generic.empty() || !TA.empty() || !TB.empty() || !PT.empty()) {
                if (nruns >= TILE_MAXRUNS) return false;
                TRunDesc& d = a->runs[nruns];
                d.kind = RUN_SLOT;
                d.s_slot = -1;
                d.ta = d.tb = d.pt = -1;
                for (int i = 0; i < TILE_T; ++i) d.ct_slot[i][0] = d.ct_slot[i][1] = -1;
                for (int j = 0; j < TILE_R; ++j) d.cr_slot[j][0] = d.cr_slot[j][1] = -1;
                std::vector<std::vector<TTerm<R>>> bucket(1 + 2 * TILE_T + 2 * TILE_R);
                uint8_t single0 = 0;
                if (!TA.empty()) {
                    d.ta = (int32_t)fac.size();
                    d.has_scalar = 1;
                    for (auto& z : TA) fac.push_back(to_r(z));
                }
                if (!TB.empty()) {
                    d.tb = (int32_t)fac.size();
                    for (auto& z : TB) fac.push_back(to_r(z));
                    for (int j = 0; j < TILE_R; ++j) {
                        bool any0 = false, any1 = false;
                        for (int tid = 0; tid < TILE_THREADS; ++tid) {
                            any0 |= TB[((size_t)tid * TILE_R + j) * 2] != cd(1, 0);
                            any1 |= TB[((size_t)tid * TILE_R + j) * 2 + 1] != cd(1, 0);
                        }
                        if (any0 || any1) d.ru |= (uint8_t)(1u << j);
                        if (any0) single0 |= (uint8_t)(1u << j);
                    }
                }
                if (!PT.empty()) {
                    d.pt = (int32_t)fac.size();
                    for (auto& z : PT) fac.push_back(to_r(z));
                }
                for (auto* ht : slotable) {
                    TTerm<R> tt;
                    std::memset(&tt, 0, sizeof(tt));
                    tt.f = to_r(ht->f);
                    const uint64_t cb = ht->mask & ~wmask, rb = ht->mask & rmask, tbm = ht->mask & wmask & ~rmask;
                    tt.cmask = cb;
                    tt.cval = ht->val & cb;
                    if (!tbm && !rb) {
                        bucket[0].push_back(tt);
                    } else if (tbm) {
                        const int b = __builtin_ctzll(tbm);
                        bucket[1 + 2 * tl_of_bit[b] + (int)((ht->val >> b) & 1)].push_back(tt);
                    } else {
                        const int b = __builtin_ctzll(rb);
                        const int vv = (int)((ht->val >> b) & 1);
                        bucket[1 + 2 * TILE_T + 2 * rl_of_bit[b] + vv].push_back(tt);
                        d.ru |= (uint8_t)(1u << rl_of_bit[b]);
                        if (!vv) single0 |= (uint8_t)(1u << rl_of_bit[b]);
                    }
                }
                for (int q = 0; q < (int)bucket.size(); ++q) {
                    if (bucket[q].empty()) continue;
                    const int sl = new_slot(bucket[q]);
                    if (q == 0) {
                        d.s_slot = (int16_t)sl;
                        d.has_scalar = 1;
                    } else if (q < 1 + 2 * TILE_T) {
                        d.ct_slot[(q - 1) >> 1][(q - 1) & 1] = (int16_t)sl;
                        d.has_scalar = 1;
                    } else {
                        const int z = q - 1 - 2 * TILE_T;
                        d.cr_slot[z >> 1][z & 1] = (int16_t)sl;
                    }
                }
                // generic L terms (rare): per-thread predicate over C|T bits
                LRange lr{nruns, lterms_all.size(), 0};
                for (auto* ht : generic) {
                    TTerm<R> tt;
                    std::memset(&tt, 0, sizeof(tt));
                    tt.f = to_r(ht->f);
                    const uint64_t cb = ht->mask & ~wmask, rb = ht->mask & rmask, tbm = ht->mask & wmask & ~rmask;
                    tt.cmask = cb | tbm;
                    tt.cval = ht->val & (cb | tbm);
                    for (int b = 0; b < 64; ++b)
                        if ((rb >> b) & 1) {
                            tt.rmask |= (uint8_t)(1u << rl_of_bit[b]);
                            if ((ht->val >> b) & 1) tt.rval |= (uint8_t)(1u << rl_of_bit[b]);
                        }
                    const int nr = popc64(rb);
                    if (nr == 0) d.has_scalar = 1;
                    if (nr == 1) {
                        d.ru |= tt.rmask;
                        if (!tt.rval) single0 |= tt.rmask;
                    }
                    lterms_all.push_back(tt);
                }
                lr.e = lterms_all.size();
                lranges.push_back(lr);
                d.r0one = (uint8_t)(d.ru & ~single0);
                TOp rop;
                std::memset(&rop, 0, sizeof(rop));
                rop.type = TO_RUN;
                rop.cx = -1;
                rop.idx = (uint16_t)nruns++;
                ops.push_back(rop);
            }
            for (auto& grp : groups) {
                if (nruns >= TILE_MAXRUNS) return false;
                const int anc = grp.first;
                TRunDesc& d = a->runs[nruns];
                d.kind = RUN_ANCHOR;
                d.anc_r = 1;
                d.anc = (uint8_t)rl_of_bit[anc];
                d.aslot[0] = d.aslot[1] = -1;
                d.fac = (uint32_t)fac.size();
                std::vector<Cx<R>> f(2 * TILE_T * 2 + 2 * TILE_R * 2, Cx<R>{(R)1, (R)0});
                std::vector<cd> fd(f.size(), cd(1, 0));
                std::vector<TTerm<R>> sl[2];
                std::vector<cd> FT;
                d.ft = -1;
                for (auto* ht : grp.second) {
                    const int vv = (int)((ht->val >> anc) & 1);
                    d.vmask |= (uint8_t)(1u << vv);
                    const uint64_t other = ht->mask & ~(1ull << anc);
                    if (!other) {
                        TTerm<R> tt;
                        std::memset(&tt, 0, sizeof(tt));
                        tt.f = to_r(ht->f);
                        sl[vv].push_back(tt);  // always-true predicate
                        continue;
                    }
                    const int b = __builtin_ctzll(other);
                    const int xb = (int)((ht->val >> b) & 1);
                    const char c = cls(b);
                    if (c == 'C') {
                        TTerm<R> tt;
                        std::memset(&tt, 0, sizeof(tt));
                        tt.f = to_r(ht->f);
                        tt.cmask = other;
                        tt.cval = ht->val & other;
                        sl[vv].push_back(tt);
                    } else if (c == 'T') {
                        if (FT.empty()) FT.assign(2 * TILE_THREADS, cd(1, 0));
                        const int i = tl_of_bit[b];
                        for (int tid = 0; tid < TILE_THREADS; ++tid)
                            if (((tid >> i) & 1) == xb) FT[vv * TILE_THREADS + tid] *= ht->f;
                    } else {
                        const int j = rl_of_bit[b];
                        fd[2 * TILE_T * 2 + (vv * TILE_R + j) * 2 + xb] *= ht->f;
                        d.rm[vv] |= (uint8_t)(1u << j);
                    }
                }
                for (int vv = 0; vv < 2; ++vv) {
                    for (int j = 0; j < TILE_R; ++j)
                        if (((d.rm[vv] >> j) & 1) && fd[2 * TILE_T * 2 + (vv * TILE_R + j) * 2] == cd(1, 0))
                            d.r1only[vv] |= (uint8_t)(1u << j);
                    if (!sl[vv].empty()) d.aslot[vv] = (int16_t)new_slot(sl[vv]);
                }
                for (size_t q = 0; q < f.size(); ++q) fac.push_back(to_r(fd[q]));
                if (!FT.empty()) {
                    d.ft = (int32_t)fac.size();
                    for (auto& z : FT) fac.push_back(to_r(z));
                }
                TOp rop;
                std::memset(&rop, 0, sizeof(rop));
                rop.type = TO_RUN;
                rop.cx = -1;
                rop.idx = (uint16_t)nruns++;
                ops.push_back(rop);
            }
        }
        a->seg[si].op1 = (uint16_t)ops.size();
    }
    if ((int)ops.size() > TILE_MAXOPS || (int)slots.size() > TILE_MAXSLOTS) return false;
    for (size_t o = 0; o < ops.size(); ++o) a->ops[o] = ops[o];
    a->nops = (int)ops.size();
    // L terms go after the slot terms; patch the ranges
    const size_t lbase = terms.size();
    for (auto& x : lterms_all) terms.push_back(x);
    for (auto& lr : lranges) {
        a->runs[lr.run].l0 = (uint16_t)(lbase + lr.b);
        a->runs[lr.run].l1 = (uint16_t)(lbase + lr.e);
    }
    if (terms.size() > 65535) return false;
    a->nslots = (int)slots.size();
    // program buffer layout
    auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
    size_t off = 0;
    a->lay.terms = (uint32_t)off;
    off = align(off + terms.size() * sizeof(TTerm<R>));
    a->lay.slots = (uint32_t)off;
    off = align(off + slots.size() * sizeof(TSlot));
    a->lay.mats = (uint32_t)off;
    off = align(off + mats.size() * sizeof(Cx<R>));
    a->lay.fac = (uint32_t)off;
    off = align(off + fac.size() * sizeof(Cx<R>));
    if (off > TileStaging::kBytes) return false;
    blob.assign(off, 0);
    if (!terms.empty()) std::memcpy(blob.data() + a->lay.terms, terms.data(), terms.size() * sizeof(TTerm<R>));
    if (!slots.empty()) std::memcpy(blob.data() + a->lay.slots, slots.data(), slots.size() * sizeof(TSlot));
    if (!mats.empty()) std::memcpy(blob.data() + a->lay.mats, mats.data(), mats.size() * sizeof(Cx<R>));
    if (!fac.empty()) std::memcpy(blob.data() + a->lay.fac, fac.data(), fac.size() * sizeof(Cx<R>));
    return true;
}

bool tile_fits(const TileSpec& t, int nl, int amp_bytes) {
    std::vector<unsigned char> blob;
    if (amp_bytes == 8) {
        static TileArgs<float>* a = new TileArgs<float>;
        return lower_tile<float>(t, nl, a, blob);
    }
    static TileArgs<double>* a = new TileArgs<double>;
    return lower_tile<double>(t, nl, a, blob);
}

template <typename R>
cudaError_t run_tile(const TileSpec& t, void* psi, int nl, cudaStream_t st, TileStaging& stg, LaunchStats& ls) {
    static TileArgs<R>* a = new TileArgs<R>;  // parameter staging (copied by the launch)
    static std::vector<unsigned char> blob;
    if (!lower_tile<R>(t, nl, a, blob)) return cudaErrorInvalidValue;
    a->psi = psi;
    cudaError_t e = stg.init();
    if (e != cudaSuccess) return e;
    const int k = stg.next;
    stg.next = (stg.next + 1) % TileStaging::kSlots;
    cudaEventSynchronize(stg.ev[k]);  // the previous copy out of this host slot is done
    unsigned char* h = stg.host + (size_t)k * TileStaging::kBytes;
    unsigned char* d = stg.dev + (size_t)k * TileStaging::kBytes;
    if (!blob.empty()) {
        std::memcpy(h, blob.data(), blob.size());
        e = cudaMemcpyAsync(d, h, blob.size(), cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return e;
    }
    e = cudaEventRecord(stg.ev[k], st);
    if (e != cudaSuccess) return e;
    a->tables = d;
    const size_t smem = sizeof(Cx<R>) * ((size_t)(1 << TILE_W) + (size_t)std::max(a->nslots, 1));
    static size_t attr = 0;
    if (smem > attr) {
        const size_t want = sizeof(Cx<R>) * ((size_t)(1 << TILE_W) + TILE_MAXSLOTS);
        e = cudaFuncSetAttribute(tile_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
        if (e != cudaSuccess) return e;
        attr = want;
    }
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t grid = std::min<uint64_t>(a->ntiles, (uint64_t)sms * 2);
    tile_kernel<R><<<(unsigned)grid, TILE_THREADS, smem, st>>>(*a);
    ls.launches++;
    return cudaGetLastError();
}

template cudaError_t run_tile<float>(const TileSpec&, void*, int, cudaStream_t, TileStaging&, LaunchStats&);
template cudaError_t run_tile<double>(const TileSpec&, void*, int, cudaStream_t, TileStaging&, LaunchStats&);

}  // namespace qj
