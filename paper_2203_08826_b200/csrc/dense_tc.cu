// dense_tc.cu -- a complex64 dense 5-qubit gate (a fused 32x32 block, the
// paper's "fusing gates up to about five [qubits]", applied
// as Eq. 1) as a tensor-core contraction on tcgen05.mma.
//
// For every group g of the 2^(n-5) groups (members m(g, j) = base(g) |
// offset(j), j = 0..31, the first-listed target being the MSB of j) the pass
// computes v' = U v.  Written over the reals, with x = (Re v_0..Re v_31,
// Im v_0..Im v_31) and o likewise for v',
//     o = A x,  A = [[Ur, -Ui], [Ui, Ur]]  (64 x 64),
// and for a tile of 128 groups as rows:  D (128 x 64) = X (128 x 64) . A^T.
// X is the MMA's A operand (M = 128 groups, K = 64), A^T its B operand
// (N = 64 outputs), D lives in tensor memory (TMEM, 64 fp32 columns per tile,
// row i on TMEM lane i), so thread i of the tile's four warps reads back the
// whole output row of its own group with one tcgen05.ld.
//
// Precision: 3xTF32.  Every fp32 operand is split x = hi + lo with hi = x
// truncated to TF32 and lo = x - hi (exact); D = Xhi.Ahi + Xhi.Alo + Xlo.Ahi
// accumulated in fp32 as one K = 192 chain of 24 MMAs (K = 8 each): relative
// error ~2^-20 per product, well inside the complex64 tolerance (R8).
//
// Data movement: each thread loads its group's 32 amplitudes (a warp's 32
// consecutive groups are consecutive addresses when the target bits are >= 5),
// writes X hi / lo into shared memory in the canonical no-swizzle K-major
// layout (8-row x 16-byte core matrices: byte offset of (row r, k) =
// (r%8)*16 + (k%4)*4 + (k/4)*128 + (r/8)*2048), one thread issues the 24 MMAs
// and commits them to an mbarrier, and the outputs go back in place.  Two
// workers (4 warps each) per CTA alternate tiles, and each prefetches its next
// tile's amplitudes into registers while its MMAs run.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "common.cuh"
#include "dense_tc.h"

namespace qj {

namespace {

constexpr int kTcRows = 128;           // groups per tile (MMA M)
constexpr int kTcWorkers = 2;          // tiles in flight per CTA
constexpr int kTcThreads = kTcRows * kTcWorkers;
constexpr uint32_t kXBytes = kTcRows * 64 * 4;  // one fp32 operand tile (32 KiB)
constexpr uint32_t kYBytes = 64 * 64 * 4;       // A^T (16 KiB)
// smem: Yhi, Ylo, then per worker Xhi, Xlo, then mbarriers and the TMEM base
constexpr size_t kTcSmem = 2 * kYBytes + kTcWorkers * 2 * kXBytes + 64;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (row, k) in the canonical no-swizzle K-major layout
__host__ __device__ __forceinline__ uint32_t kmaj(uint32_t row, uint32_t k) {
    return (row & 7) * 16 + (k & 3) * 4 + (k >> 2) * 128 + (row >> 3) * 2048;
}

__device__ __forceinline__ float tf32_hi(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// UMMA shared-memory matrix descriptor: no swizzle, K-major, LBO = 128 B
// (adjacent core matrices along K), SBO = 2048 B (adjacent 8-row groups),
// version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(2048u >> 4) << 32) |
           (1ull << 46);
}

// instruction descriptor: kind::tf32, D fp32, A/B TF32 K-major, N = 64, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(dtmem),
        "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_addr(bar);
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float (&o)[64]) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,"
        "%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,"
        "%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
          "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
          "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
          "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
          "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) o[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ uint64_t group_base(uint64_t g, const TcArgs& a) {
    uint64_t x = g;
    for (int i = 0; i < a.nins; ++i) x = insert_zero(x, a.ins_pos[i]);
    return x | a.fix_val;
}

constexpr int kStageStride = 33;  // float2 per staged row (32 members + 1 pad: 2-way bank conflicts at most)

template <bool STAGED>
__global__ void __launch_bounds__(kTcThreads, 1) dense5_tc_kernel(const __grid_constant__ TcArgs a) {
    extern __shared__ __align__(1024) unsigned char smraw[];
    unsigned char* yhi = smraw;
    unsigned char* ylo = smraw + kYBytes;
    const int wk = threadIdx.x / kTcRows, row = threadIdx.x % kTcRows;
    unsigned char* xhi = smraw + 2 * kYBytes + (size_t)wk * 2 * kXBytes;
    unsigned char* xlo = xhi + kXBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + 2 * kYBytes + (size_t)kTcWorkers * 2 * kXBytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + kTcWorkers);
    const int warp = threadIdx.x / 32;

    // TMEM: 64 fp32 columns per worker
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(tmem_slot)),
                     "r"(64u * kTcWorkers)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    // B operand A^T (rows n = outputs, K = inputs, K-major), split hi / lo
    for (int idx = threadIdx.x; idx < 64 * 64; idx += kTcThreads) {
        const int n = idx >> 6, k = idx & 63;
        const float2 u = a.u[n & 31][k & 31];
        float v;
        if (n < 32) v = k < 32 ? u.x : -u.y;  // rows 0..31: Re(v'_n) = sum Ur x_re - Ui x_im
        else v = k < 32 ? u.y : u.x;          // rows 32..63: Im(v'_n) = sum Ui x_re + Ur x_im
        const float h = tf32_hi(v);
        *reinterpret_cast<float*>(yhi + kmaj(n, k)) = h;
        *reinterpret_cast<float*>(ylo + kmaj(n, k)) = v - h;
    }
    if (threadIdx.x == 0) {
        for (int w = 0; w < kTcWorkers; ++w) mbar_init1(&bars[w]);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *tmem_slot + (uint32_t)(wk * 64);                 // this worker's columns
    const uint32_t tload = tmem + ((uint32_t)((warp & 3) * 32) << 16);      // this warp's lanes
    const uint32_t sxhi = smem_addr(xhi), sxlo = smem_addr(xlo), syhi = smem_addr(yhi), sylo = smem_addr(ylo);

    const uint64_t ntiles = a.ngroups / kTcRows;
    float2* psi = static_cast<float2*>(a.psi);
    float2 v[32];
    uint64_t t = (uint64_t)blockIdx.x * kTcWorkers + wk;
    const uint64_t tstep = (uint64_t)gridDim.x * kTcWorkers;
    uint64_t base = 0;
    // staged form: this thread's share of every tile is L = row + 128 m
    float2* stage = reinterpret_cast<float2*>(xhi);  // aliases X hi / lo (free between MMAs)
    uint64_t arow = 0;
    uint32_t srow = 0;
    if constexpr (STAGED) {
        for (int i = 0; i < 7; ++i)
            if ((row >> i) & 1) {
                arow |= 1ull << a.lpos_row[i];
                srow += a.w_row[i];
            }
    }
    // (staged form: the next tile's amplitudes are loaded coalesced into v in
    // L order while the MMAs run, and redistributed to rows through shared
    // memory at the start of the tile)
    auto load_tile = [&](uint64_t tt) {
        if constexpr (STAGED) {
            const uint64_t tb = group_base(tt * kTcRows, a) | arow;
#pragma unroll
            for (int m = 0; m < 32; ++m) v[m] = __ldcs(psi + (tb | a.addr_m[m]));
        } else {
            base = group_base(tt * kTcRows + row, a);
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __ldcs(psi + base + a.moff[j]);
        }
    };
    if (t < ntiles) load_tile(t);
    uint32_t phase = 0;
    for (; t < ntiles; t += tstep, phase ^= 1) {
        if constexpr (STAGED) {  // L order -> rows
#pragma unroll
            for (int m = 0; m < 32; ++m) stage[srow + a.sidx_m[m]] = v[m];
            asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wk), "r"(kTcRows) : "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = stage[row * kStageStride + j];
            asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wk), "r"(kTcRows) : "memory");  // staging free for X
        }
        // X hi / lo of this thread's group (row): K = (Re v_0..31, Im v_0..31)
#pragma unroll
        for (int c = 0; c < 16; ++c) {  // 4 consecutive k per 16-byte store
            float4 h, l;
            float e[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int k = 4 * c + q;
                e[q] = k < 32 ? v[k].x : v[k - 32].y;
            }
            h = make_float4(tf32_hi(e[0]), tf32_hi(e[1]), tf32_hi(e[2]), tf32_hi(e[3]));
            l = make_float4(e[0] - h.x, e[1] - h.y, e[2] - h.z, e[3] - h.w);
            *reinterpret_cast<float4*>(xhi + kmaj(row, 4 * c)) = h;
            *reinterpret_cast<float4*>(xlo + kmaj(row, 4 * c)) = l;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");      // generic writes -> MMA reads
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");  // last tile's TMEM reads done
        asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wk), "r"(kTcRows) : "memory");
        if (row == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)  // Xhi . Ahi
                mma_tf32(tmem, sdesc(sxhi + ks * 256), sdesc(syhi + ks * 256), ks > 0);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)  // + Xhi . Alo
                mma_tf32(tmem, sdesc(sxhi + ks * 256), sdesc(sylo + ks * 256), 1);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)  // + Xlo . Ahi
                mma_tf32(tmem, sdesc(sxlo + ks * 256), sdesc(syhi + ks * 256), 1);
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                             smem_addr(&bars[wk]))
                         : "memory");
        }
        // prefetch the next tile's amplitudes while the MMAs run
        const uint64_t cur = base;
        const uint64_t tn = t + tstep;
        if (tn < ntiles) load_tile(tn);
        mbar_wait_parity(&bars[wk], phase);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        float o[64];
        tmem_ld64(tload, o);
        if constexpr (STAGED) {  // rows -> staging -> cooperative coalesced stores
#pragma unroll
            for (int j = 0; j < 32; ++j) stage[row * kStageStride + j] = make_float2(o[j], o[32 + j]);
            asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wk), "r"(kTcRows) : "memory");
            const uint64_t tb = group_base(t * kTcRows, a) | arow;
#pragma unroll 8
            for (int m = 0; m < 32; ++m) __stcs(psi + (tb | a.addr_m[m]), stage[srow + a.sidx_m[m]]);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // staging (X) is rewritten next tile
            asm volatile("bar.sync %0, %1;\n" ::"r"(1 + wk), "r"(kTcRows) : "memory");
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcs(psi + cur + a.moff[j], make_float2(o[j], o[32 + j]));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(*tmem_slot), "r"(64u * kTcWorkers)
                     : "memory");
    }
}

}  // namespace

bool dense_tc_enabled() {
    static const bool on = !(getenv("QJ_TC") && getenv("QJ_TC")[0] == '0');
    return on;
}

bool dense_tc_supports(const Pass& p, int nl) {
    if (p.kind != PK_DENSE || p.k != 5 || p.touch != 0xffffffffu) return false;
    return nl - 5 - p.nfix >= 7 + 0 && (1ull << (nl - 5 - p.nfix)) >= (uint64_t)kTcRows;
}

cudaError_t run_dense_tc(const Pass& p, void* psi, int nl, cudaStream_t st, LaunchStats& ls) {
    static TcArgs* a = new TcArgs;
    std::memset(a, 0, sizeof(TcArgs));
    a->psi = psi;
    for (int r = 0; r < 32; ++r)
        for (int c = 0; c < 32; ++c) {
            const cd z = p.m[(size_t)r * 32 + c];
            a->u[r][c] = make_float2((float)z.real(), (float)z.imag());
        }
    for (int j = 0; j < 32; ++j) {
        uint64_t off = 0;
        for (int i = 0; i < 5; ++i)
            if ((j >> (4 - i)) & 1) off |= 1ull << p.tpos[i];
        a->moff[j] = off;
    }
    int pos[QJ_MAX_TARGETS + 64];
    int np = 0;
    for (int i = 0; i < 5; ++i) pos[np++] = p.tpos[i];
    for (int i = 0; i < p.nfix; ++i) {
        pos[np++] = p.fpos[i];
        if (p.fval[i]) a->fix_val |= 1ull << p.fpos[i];
    }
    std::sort(pos, pos + np);
    if (np > 16) return cudaErrorInvalidValue;
    a->nins = np;
    for (int i = 0; i < np; ++i) a->ins_pos[i] = pos[i];
    a->ngroups = 1ull << (nl - np);
    // staged when a thread's own 32 members would not be coalesced across a warp
    // (some target or fixed bit below bit 5: the warp's groups are not 32
    // consecutive amplitudes)
    a->staged = pos[0] < 5 ? 1 : 0;
    if (a->staged) {
        int lpos[12], ltype[12], nlp = 0, k = 0;  // ltype: 0..6 group bit k, 100 + t target t
        for (int b = 0; nlp < 12 && b < nl; ++b) {
            bool ins = false;
            for (int i = 0; i < np; ++i) ins |= pos[i] == b;
            int tt = -1;
            for (int i = 0; i < 5; ++i)
                if (p.tpos[i] == b) tt = i;
            if (tt >= 0) {
                lpos[nlp] = b;
                ltype[nlp++] = 100 + tt;
            } else if (!ins && k < 7) {
                lpos[nlp] = b;
                ltype[nlp++] = k++;
            }
        }
        if (nlp != 12) return cudaErrorInvalidValue;
        auto weight = [&](int i) -> uint32_t {
            return ltype[i] >= 100 ? (1u << (4 - (ltype[i] - 100))) : (uint32_t)kStageStride << ltype[i];
        };
        for (int i = 0; i < 7; ++i) {
            a->lpos_row[i] = lpos[i];
            a->w_row[i] = weight(i);
        }
        for (int m = 0; m < 32; ++m) {
            uint64_t ad = 0;
            uint32_t sx = 0;
            for (int i = 0; i < 5; ++i)
                if ((m >> i) & 1) {
                    ad |= 1ull << lpos[7 + i];
                    sx += weight(7 + i);
                }
            a->addr_m[m] = ad;
            a->sidx_m[m] = sx;
        }
    }
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(dense5_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(dense5_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTcSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const uint64_t ntiles = a->ngroups / kTcRows;
    const uint64_t grid = std::min<uint64_t>((ntiles + kTcWorkers - 1) / kTcWorkers, (uint64_t)device_sms());
    if (a->staged) dense5_tc_kernel<true><<<(unsigned)grid, kTcThreads, kTcSmem, st>>>(*a);
    else dense5_tc_kernel<false><<<(unsigned)grid, kTcThreads, kTcSmem, st>>>(*a);
    ls.launches++;
    return cudaGetLastError();
}

}  // namespace qj
