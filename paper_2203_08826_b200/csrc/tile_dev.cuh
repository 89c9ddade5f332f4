// tile_dev.cuh -- device side of the fused window tile pass (tile.h): the
// register-level gate ops, the phase runs, the tile phases (load, SMEM
// transpose, store) and the ahead-of-time interpreter kernel.  Compiled by
// nvcc into libqj and, unchanged, by NVRTC as the prelude of every
// circuit-specialised tile kernel (tile_jit.cpp), which calls the same
// functions with every operand as a compile-time constant.
#pragma once

#include "tile_abi.h"

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
    return i ^ (((i >> 3) ^ (i >> 6) ^ (i >> 9) ^ (i >> 12)) & 7u);
}
template <>
__host__ __device__ __forceinline__ uint32_t swz<float>(uint32_t i) {
    return i ^ (((i >> 4) ^ (i >> 8) ^ (i >> 12)) & 15u);
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

// Unscaled Hadamard butterfly (x + y, x - y): the JIT kernels apply the
// product of the pass's 1/sqrt(2) factors once, at the store.
template <typename R, int A>
__device__ __forceinline__ void op_hu(Cx<R> (&v)[TILE_NREG]) {
#pragma unroll
    for (int j = 0; j < TILE_NREG / 2; ++j) {
        const int lo = ((j >> A) << (A + 1)) | (j & ((1 << A) - 1));
        const int hi = lo | (1 << A);
        const Cx<R> x = v[lo], y = v[hi];
        v[lo] = Cx<R>{x.re + y.re, x.im + y.im};
        v[hi] = Cx<R>{x.re - y.re, x.im - y.im};
    }
}

template <typename R>
__device__ __forceinline__ void scale_all(Cx<R> (&v)[TILE_NREG], R s) {
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) v[r] = Cx<R>{v[r].re * s, v[r].im * s};
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

// cfma with the matrix entry's zero components known at compile time
// (NZ bit 0: re != 0, bit 1: im != 0); JIT kernels specialise U1 / U2 ops on
// the zero pattern of their matrices (RX / RY / fSim are half zeros), the
// values stay runtime data.  Same FMA order as cfma on the nonzero terms.
template <typename R, int NZ>
__device__ __forceinline__ void cfma_nz(Cx<R>& acc, Cx<R> a, Cx<R> b) {
    if constexpr (NZ & 1) acc.re = fma(a.re, b.re, acc.re);
    if constexpr (NZ & 2) acc.re = fma(-a.im, b.im, acc.re);
    if constexpr (NZ & 1) acc.im = fma(a.re, b.im, acc.im);
    if constexpr (NZ & 2) acc.im = fma(a.im, b.re, acc.im);
}

template <typename R, int A, bool C, uint32_t NZ>
__device__ __forceinline__ void op_u1_nz(Cx<R> (&v)[TILE_NREG], const Cx<R>* m, uint32_t crm, uint32_t crv, bool ok) {
    const Cx<R> m00 = m[0], m01 = m[1], m10 = m[2], m11 = m[3];
#pragma unroll
    for (int j = 0; j < TILE_NREG / 2; ++j) {
        const int lo = ((j >> A) << (A + 1)) | (j & ((1 << A) - 1));
        const int hi = lo | (1 << A);
        if (!C || (ok && ((uint32_t)lo & crm) == crv)) {
            const Cx<R> x = v[lo], y = v[hi];
            Cx<R> o0{R(0), R(0)}, o1{R(0), R(0)};
            cfma_nz<R, (NZ >> 0) & 3>(o0, m00, x);
            cfma_nz<R, (NZ >> 2) & 3>(o0, m01, y);
            cfma_nz<R, (NZ >> 4) & 3>(o1, m10, x);
            cfma_nz<R, (NZ >> 6) & 3>(o1, m11, y);
            v[lo] = o0;
            v[hi] = o1;
        }
    }
}

// 4x4 on register bits A (matrix MSB) and B, zero pattern NZ (2 bits per entry, row-major)
template <typename R, int A, int B, bool C, uint32_t NZ>
__device__ __forceinline__ void op_u2_nz(Cx<R> (&v)[TILE_NREG], const Cx<R>* m, uint32_t crm, uint32_t crv, bool ok) {
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
            for (int c = 0; c < 4; ++c) {
                constexpr uint32_t dummy = 0;
                (void)dummy;
                switch ((NZ >> (2 * (r * 4 + c))) & 3) {
                    case 1: cfma_nz<R, 1>(o, m[r * 4 + c], in[c]); break;
                    case 2: cfma_nz<R, 2>(o, m[r * 4 + c], in[c]); break;
                    case 3: cfma_nz<R, 3>(o, m[r * 4 + c], in[c]); break;
                    default: break;
                }
            }
            v[id[r]] = o;
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

template <typename R, int ANC, int VAL, int J = 0>
__device__ __forceinline__ void mul_pairs(Cx<R> (&v)[TILE_NREG], const Cx<R> (&g)[TILE_R][2], uint32_t use,
                                          uint32_t only1) {
    if constexpr (J < TILE_R) {
        if (((use >> J) & 1) && ANC != J) mul_pair<R, ANC, VAL, J>(v, g[J][0], g[J][1], (only1 >> J) & 1);
        mul_pairs<R, ANC, VAL, J + 1>(v, g, use, only1);
    }
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
                case 0: if constexpr (0 < TILE_R) { op_h<R, 0, false>(v, hs, crm, crv, ok); } break;
                case 1: if constexpr (1 < TILE_R) { op_h<R, 1, false>(v, hs, crm, crv, ok); } break;
                case 2: if constexpr (2 < TILE_R) { op_h<R, 2, false>(v, hs, crm, crv, ok); } break;
                case 3: if constexpr (3 < TILE_R) { op_h<R, 3, false>(v, hs, crm, crv, ok); } break;
            }
            break;
        }
        case TO_U1: {
            const Cx<R>* m = mats + op.idx;
            switch (op.a) {
                case 0: if constexpr (0 < TILE_R) { op_u1<R, 0, C>(v, m, crm, crv, ok); } break;
                case 1: if constexpr (1 < TILE_R) { op_u1<R, 1, C>(v, m, crm, crv, ok); } break;
                case 2: if constexpr (2 < TILE_R) { op_u1<R, 2, C>(v, m, crm, crv, ok); } break;
                case 3: if constexpr (3 < TILE_R) { op_u1<R, 3, C>(v, m, crm, crv, ok); } break;
            }
            break;
        }
        case TO_X:
            switch (op.a) {
                case 0: if constexpr (0 < TILE_R) { op_x<R, 0, C>(v, crm, crv, ok); } break;
                case 1: if constexpr (1 < TILE_R) { op_x<R, 1, C>(v, crm, crv, ok); } break;
                case 2: if constexpr (2 < TILE_R) { op_x<R, 2, C>(v, crm, crv, ok); } break;
                case 3: if constexpr (3 < TILE_R) { op_x<R, 3, C>(v, crm, crv, ok); } break;
            }
            break;
        case TO_U2: {
            const Cx<R>* m = mats + op.idx;
            switch (op.a * 4 + op.b) {
                case 1: if constexpr (0 < TILE_R && 1 < TILE_R) { op_u2<R, 0, 1, C>(v, m, crm, crv, ok); } break;
                case 2: if constexpr (0 < TILE_R && 2 < TILE_R) { op_u2<R, 0, 2, C>(v, m, crm, crv, ok); } break;
                case 3: if constexpr (0 < TILE_R && 3 < TILE_R) { op_u2<R, 0, 3, C>(v, m, crm, crv, ok); } break;
                case 4: if constexpr (1 < TILE_R && 0 < TILE_R) { op_u2<R, 1, 0, C>(v, m, crm, crv, ok); } break;
                case 6: if constexpr (1 < TILE_R && 2 < TILE_R) { op_u2<R, 1, 2, C>(v, m, crm, crv, ok); } break;
                case 7: if constexpr (1 < TILE_R && 3 < TILE_R) { op_u2<R, 1, 3, C>(v, m, crm, crv, ok); } break;
                case 8: if constexpr (2 < TILE_R && 0 < TILE_R) { op_u2<R, 2, 0, C>(v, m, crm, crv, ok); } break;
                case 9: if constexpr (2 < TILE_R && 1 < TILE_R) { op_u2<R, 2, 1, C>(v, m, crm, crv, ok); } break;
                case 11: if constexpr (2 < TILE_R && 3 < TILE_R) { op_u2<R, 2, 3, C>(v, m, crm, crv, ok); } break;
                case 12: if constexpr (3 < TILE_R && 0 < TILE_R) { op_u2<R, 3, 0, C>(v, m, crm, crv, ok); } break;
                case 13: if constexpr (3 < TILE_R && 1 < TILE_R) { op_u2<R, 3, 1, C>(v, m, crm, crv, ok); } break;
                case 14: if constexpr (3 < TILE_R) { op_u2<R, 3, 2, C>(v, m, crm, crv, ok); } break;
            }
            break;
        }
        case TO_SWAP: {
            const int lo = op.a < op.b ? op.a : op.b, hi = op.a < op.b ? op.b : op.a;
            switch (lo * 4 + hi) {
                case 1: if constexpr (1 < TILE_R && 0 < TILE_R) { op_swap<R, 1, 0, C>(v, crm, crv, ok); } break;
                case 2: if constexpr (2 < TILE_R && 0 < TILE_R) { op_swap<R, 2, 0, C>(v, crm, crv, ok); } break;
                case 3: if constexpr (3 < TILE_R && 0 < TILE_R) { op_swap<R, 3, 0, C>(v, crm, crv, ok); } break;
                case 6: if constexpr (2 < TILE_R && 1 < TILE_R) { op_swap<R, 2, 1, C>(v, crm, crv, ok); } break;
                case 7: if constexpr (3 < TILE_R && 1 < TILE_R) { op_swap<R, 3, 1, C>(v, crm, crv, ok); } break;
                case 11: if constexpr (3 < TILE_R) { op_swap<R, 3, 2, C>(v, crm, crv, ok); } break;
            }
            break;
        }
        default: {
            const TRunDesc& d = a.runs[op.idx];
            if (d.kind == RUN_ANCHOR) {
                switch (d.anc) {
                    case 0: if constexpr (0 < TILE_R) { anchor_run<R, 0>(a, d, v, tid, tab); } break;
                    case 1: if constexpr (1 < TILE_R) { anchor_run<R, 1>(a, d, v, tid, tab); } break;
                    case 2: if constexpr (2 < TILE_R) { anchor_run<R, 2>(a, d, v, tid, tab); } break;
                    case 3: if constexpr (3 < TILE_R) { anchor_run<R, 3>(a, d, v, tid, tab); } break;
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
    uint64_t x = 0;
#pragma unroll
    for (int c = 0; c < TILE_TCH; ++c) x |= a.tph[s][c][(tid >> (4 * c)) & 15];
    return x;
}
// ... of the last segment's stores (output permutation applied)
template <typename R>
__device__ __forceinline__ uint64_t thread_phys_out(const TileArgs<R>& a, int tid) {
    uint64_t x = 0;
#pragma unroll
    for (int c = 0; c < TILE_TCH; ++c) x |= a.tph_out[c][(tid >> (4 * c)) & 15];
    return x;
}
template <typename R>
__device__ __forceinline__ uint32_t thread_loc(const TileArgs<R>& a, int s, int tid) {
    uint32_t x = 0;
#pragma unroll
    for (int c = 0; c < TILE_TCH; ++c) x |= a.tlo[s][c][(tid >> (4 * c)) & 15];
    return x;
}

// ---------------------------------------------------------------- tile phases
// Per-tile base index (non-window bits of `tile`) and the per-tile products of
// the tile-dependent phase terms (slots) into SMEM.
// Slot products of one tile: warp w fills slots w, w + warps, ...; its lanes
// take every 32nd term of the slot (independent loads, no dependent chain) and
// a fixed xor-butterfly multiplies the 32 partial products, so the result is
// deterministic and the same in every kernel flavour.
template <typename R>
__device__ __forceinline__ void tile_slots(const TileArgs<R>& a, uint64_t tg, Cx<R>* tab, int tid) {
    const TSlot* slots = reinterpret_cast<const TSlot*>(a.tables + a.lay.slots);
    const TTerm<R>* terms = reinterpret_cast<const TTerm<R>*>(a.tables + a.lay.terms);
    const int lane = tid & 31;
    for (int e = tid >> 5; e < a.nslots; e += TILE_THREADS / 32) {
        const TSlot sl = slots[e];
        Cx<R> p = cone<R>();
        for (uint32_t t = sl.t0 + lane; t < sl.t1; t += 32)
            if ((tg & terms[t].cmask) == terms[t].cval) p = cmul(p, terms[t].f);
#pragma unroll
        for (int o = 16; o; o >>= 1) p = cmul(p, shfl_xor(p, o));
        if (lane == 0) tab[e] = p;
    }
}

// JIT kernels stage the slot terms (predicate + factor) and slot ranges in
// shared memory once per CTA, so the per-tile products read no global memory.
template <typename R>
struct STerm {
    uint64_t cmask, cval;
    Cx<R> f;
};
template <typename R>
__device__ __forceinline__ void tile_slots_staged(const STerm<R>* terms, const TSlot* slots, int nslots, uint64_t tg,
                                                  Cx<R>* tab, int tid) {
    const int lane = tid & 31;
    for (int e = tid >> 5; e < nslots; e += TILE_THREADS / 32) {
        const TSlot sl = slots[e];
        Cx<R> p = cone<R>();
        for (uint32_t t = sl.t0 + lane; t < sl.t1; t += 32)
            if ((tg & terms[t].cmask) == terms[t].cval) p = cmul(p, terms[t].f);
#pragma unroll
        for (int o = 16; o; o >>= 1) p = cmul(p, shfl_xor(p, o));
        if (lane == 0) tab[e] = p;
    }
}

template <typename R>
__device__ __forceinline__ uint64_t tile_begin(const TileArgs<R>& a, uint64_t tile, Cx<R>* tab, int tid) {
    uint64_t tb = tile;
#pragma unroll
    for (int i = 0; i < TILE_W; ++i) tb = insert_zero(tb, a.wpos[i]);
    tile_slots(a, tb | a.gbase, tab, tid);  // predicates see the global bits too
    return tb;
}

// JIT kernels address the tile with compile-time register offsets: one
// amplitude copy / store at element offset `off` from a per-thread base.
template <typename R>
__device__ __forceinline__ void cp_amp(Cx<R>* s, const Cx<R>* g);
template <typename R>
__device__ __forceinline__ void st_amp(Cx<R>* g, Cx<R> v) {
    store_amp(g, 0, v);
}

// HBM <-> registers with the mapping of segment s (s = 0 loads, s = last stores).
template <typename R>
__device__ __forceinline__ void tile_load(const TileArgs<R>& a, int s, Cx<R> (&v)[TILE_NREG], uint64_t tb, int tid) {
    const TSeg& S = a.seg[s];
    const uint64_t base = tb | thread_phys(a, s, tid);
    uint64_t rm[TILE_R];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j) rm[j] = 1ull << a.wpos[S.rbits[j]];
    const Cx<R>* psi = reinterpret_cast<const Cx<R>*>(a.psi);
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) {
        uint64_t x = base;
#pragma unroll
        for (int j = 0; j < TILE_R; ++j)
            if ((r >> j) & 1) x |= rm[j];
        v[r] = load_amp(psi, x);
    }
}
template <typename R>
__device__ __forceinline__ void tile_store(const TileArgs<R>& a, int s, const Cx<R> (&v)[TILE_NREG], uint64_t tb,
                                           int tid) {
    const TSeg& S = a.seg[s];
    const uint64_t base = tb | thread_phys_out(a, tid);  // (the last segment: s == nseg - 1)
    uint64_t rm[TILE_R];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j) rm[j] = 1ull << a.wpos[a.operm[S.rbits[j]]];
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) {
        uint64_t x = base;
#pragma unroll
        for (int j = 0; j < TILE_R; ++j)
            if ((r >> j) & 1) x |= rm[j];
        store_amp(a.psi, x, v[r]);
    }
}

// Asynchronous prefetch of a tile into the (swizzled) SMEM buffer with the
// mapping of segment 0, and the matching register load.  The JIT kernels issue
// the prefetch of tile i+1 right after tile i's last transpose, so its HBM
// latency overlaps the last segment's compute and the stores.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait_n() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Issue the prefetch of `tile` into `sm` (no commit: the caller groups it).
template <typename R>
__device__ __forceinline__ void tile_prefetch_issue(const TileArgs<R>& a, uint64_t tile, Cx<R>* sm, int tid) {
    uint64_t tb = tile;
#pragma unroll
    for (int i = 0; i < TILE_W; ++i) tb = insert_zero(tb, a.wpos[i]);
    const TSeg& S = a.seg[0];
    const uint64_t base = tb | thread_phys(a, 0, tid);
    const uint32_t bl = swz<R>(thread_loc(a, 0, tid));
    uint64_t rm[TILE_R];
    uint32_t sl[TILE_R];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j) {
        rm[j] = 1ull << a.wpos[S.rbits[j]];
        sl[j] = swz<R>(1u << S.rbits[j]);
    }
    const Cx<R>* psi = reinterpret_cast<const Cx<R>*>(a.psi);
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) {
        uint64_t x = base;
        uint32_t y = bl;
#pragma unroll
        for (int j = 0; j < TILE_R; ++j)
            if ((r >> j) & 1) {
                x |= rm[j];
                y ^= sl[j];
            }
        if constexpr (sizeof(R) == 8) cp_async16(sm + y, psi + x);
        else cp_async8(sm + y, psi + x);
    }
}

template <>
__device__ __forceinline__ void cp_amp<double>(Cx<double>* s, const Cx<double>* g) {
    cp_async16(s, g);
}
template <>
__device__ __forceinline__ void cp_amp<float>(Cx<float>* s, const Cx<float>* g) {
    cp_async8(s, g);
}

// Bounds check of a global amplitude pointer (checked JIT kernels only).
template <typename R>
__device__ __forceinline__ bool qj_chk(const TileArgs<R>& a, const Cx<R>* p, uint64_t count = 1) {
    const uint64_t off = (uint64_t)(p - reinterpret_cast<const Cx<R>*>(a.psi));
    if (off < a.namps && count <= a.namps - off) return true;
    if (a.chk) atomicOr(a.chk, 1u);
    return false;
}

// ---------------------------------------------------------------- ring form (TMA)
// JIT kernels in the ring form run two workers (256 threads each) per CTA over
// a ring of tile buffers filled by bulk asynchronous copies (TMA engine,
// cp.async.bulk) that complete on one mbarrier per buffer; a worker
// synchronises its own 256 threads with a named barrier.
// Programmatic dependent launch (the JIT kernels are launched with it): let
// the next pass be scheduled once every CTA of this one is resident, then
// wait until the previous grid has completed and its writes are visible.
// Everything before this call touches only host-written tables and SMEM.
__device__ __forceinline__ void grid_dep_sync() {
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

__device__ __forceinline__ void worker_sync(int wk) {
    asm volatile("bar.sync %0, 256;\n" ::"r"(1 + wk) : "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
// generic-proxy accesses of a buffer before the async proxy (TMA) writes it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// global -> shared bulk copy (16-byte multiple), completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

template <typename R>
__device__ __forceinline__ void tile_prefetch(const TileArgs<R>& a, uint64_t tile, Cx<R>* sm, int tid) {
    tile_prefetch_issue(a, tile, sm, tid);
    cp_async_commit();
}

// Ring variant: tile i's data was committed as its own cp.async group; at most
// N newer groups may still be in flight.
template <int N, typename R>
__device__ __forceinline__ void tile_load_ring(const TileArgs<R>& a, Cx<R> (&v)[TILE_NREG], const Cx<R>* sm, int tid) {
    cp_async_wait_n<N>();
    __syncthreads();
    const TSeg& S = a.seg[0];
    const uint32_t bl = swz<R>(thread_loc(a, 0, tid));
    uint32_t sl[TILE_R];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j) sl[j] = swz<R>(1u << S.rbits[j]);
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) {
        uint32_t y = bl;
#pragma unroll
        for (int j = 0; j < TILE_R; ++j)
            if ((r >> j) & 1) y ^= sl[j];
        v[r] = sm[y];
    }
}

template <typename R>
__device__ __forceinline__ void tile_load_prefetched(const TileArgs<R>& a, Cx<R> (&v)[TILE_NREG], const Cx<R>* sm,
                                                     int tid) {
    cp_async_wait_all();
    __syncthreads();
    const TSeg& S = a.seg[0];
    const uint32_t bl = swz<R>(thread_loc(a, 0, tid));
    uint32_t sl[TILE_R];
#pragma unroll
    for (int j = 0; j < TILE_R; ++j) sl[j] = swz<R>(1u << S.rbits[j]);
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) {
        uint32_t y = bl;
#pragma unroll
        for (int j = 0; j < TILE_R; ++j)
            if ((r >> j) & 1) y ^= sl[j];
        v[r] = sm[y];
    }
}

// qj_simulate: the first pass synthesises |basis> (no HBM read) ...
template <typename R>
__device__ __forceinline__ void tile_synth(const TileArgs<R>& a, Cx<R> (&v)[TILE_NREG], uint64_t tb, int tid) {
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
        v[r] = Cx<R>{x == a.synth ? R(1) : R(0), R(0)};
    }
}

// ... and the last pass accumulates the marginal of the listed physical bits
// (bin = tile part | thread part | register part, disjoint bit sets).
__device__ __forceinline__ uint32_t bin_of(uint64_t x, const int8_t* pos, int nq) {
    uint32_t b = 0;
    for (int k = 0; k < nq; ++k) b = (b << 1) | (uint32_t)((x >> pos[k]) & 1u);
    return b;
}
// Fused marginal, readout bits all inside the window: bin(thread, r) is
// tile-independent, so each thread accumulates |v_r|^2 into its own SMEM slot
// acc[r][tid] (no atomics); tile_bins_flush reduces them at the end.
template <typename R>
__device__ __forceinline__ void tile_bins(const Cx<R> (&v)[TILE_NREG], double* acc, int tid) {
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r)
        acc[r * TILE_THREADS + tid] += (double)v[r].re * (double)v[r].re + (double)v[r].im * (double)v[r].im;
}
template <typename R>
__device__ __forceinline__ void tile_bins_flush(const TileArgs<R>& a, const double* acc, double* sb, uint32_t thbin,
                                                int tid) {
    const int nb = 1 << a.nbq;
    for (int i = tid; i < nb; i += TILE_THREADS) sb[i] = 0.0;
    __syncthreads();
#pragma unroll
    for (int r = 0; r < TILE_NREG; ++r) atomicAdd(&sb[thbin | a.regbin[r]], acc[r * TILE_THREADS + tid]);
    __syncthreads();
    for (int i = tid; i < nb; i += TILE_THREADS)
        if (sb[i] != 0.0) atomicAdd(&a.bins[i], sb[i]);
}

// Registers of segment s-1 -> swizzled SMEM -> registers of segment s.
template <typename R>
__device__ __forceinline__ void tile_transpose(const TileArgs<R>& a, int s, Cx<R> (&v)[TILE_NREG], Cx<R>* sm,
                                               int tid) {
    const TSeg& P = a.seg[s - 1];
    const TSeg& S = a.seg[s];
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

// The ahead-of-time interpreter: ops decoded from the parameter block.
template <typename R>
__global__ void __launch_bounds__(TILE_THREADS, TILE_MINBLOCKS) tile_kernel(const __grid_constant__ TileArgs<R> a) {
    extern __shared__ __align__(16) unsigned char smraw[];
    Cx<R>* sm = reinterpret_cast<Cx<R>*>(smraw);
    Cx<R>* tab = sm + (1 << TILE_W);
    const int tid = threadIdx.x;
    for (uint64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const uint64_t tb = tile_begin(a, tile, tab, tid);
        Cx<R> v[TILE_NREG];
        tile_load(a, 0, v, tb, tid);
        __syncthreads();  // tab ready
        for (int s = 0; s < a.nseg; ++s) {
            if (s > 0) tile_transpose(a, s, v, sm, tid);
            const uint64_t tfull = tb | a.gbase | thread_phys(a, s, tid);
            for (int o = a.seg[s].op0; o < a.seg[s].op1; ++o) apply_op(a, a.ops[o], v, tfull, tid, tab);
        }
        tile_store(a, a.nseg - 1, v, tb, tid);
        __syncthreads();  // tab / smem reuse by the next tile
    }
}

}  // namespace qj
