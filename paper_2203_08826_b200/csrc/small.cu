// small.cu -- the whole-state SMEM pass (see small.h).
//
// Each op is one planned Pass (Eq. 1 on k targets with fixed
// control / pattern bits, or a specialised X / SWAP / diagonal / phase / sign
// form): the 2^(n-k-nfix) groups are enumerated by bit
// insertion and spread over the block's threads; a barrier
// separates ops.  Roofline: launch latency + barrier latency per op (the
// state is read and written once per launch: 2 s 2^n bytes).
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "small.h"

namespace qj {
namespace {

constexpr int kSmallThreads = 512;

struct SOp {
    int32_t kind, k, nins, pad;
    uint32_t touch, data;  // data: offset of the op's coefficients in the data array
    uint64_t fval;         // fixed-bit values, positioned
    int8_t tpos[8];        // targets, matrix order (first = MSB of the member index)
    int8_t ins[24];        // targets and fixed bits, ascending (bit insertion)
};
static_assert(sizeof(SOp) == 64, "SOp layout");

// A run of consecutive diagonal passes (DIAG k <= 4, PHASE, NEG) lowers to one
// op: they commute and touch each amplitude in place, so no barrier is needed
// between them -- every thread multiplies its amplitudes by each member's
// factor (1 where the member's fixed bits do not match).
constexpr int PK_DRUN = 16;
constexpr int kMaxRun = 48;
struct DSub {
    uint64_t fmask, fval;  // fixed (control / pattern) bits that must match
    int32_t kind, k;       // PK_DIAG (k targets), PK_PHASE, PK_NEG
    uint32_t coff;         // byte offset of the coefficients in the chunk data
    int8_t tpos[4];
};
static_assert(sizeof(DSub) == 32, "DSub layout");

template <int K>
__device__ __forceinline__ void member_offsets(const SOp& op, uint32_t (&off)[1 << K]) {
#pragma unroll
    for (int m = 0; m < (1 << K); ++m) {
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) v |= ((uint32_t)(m >> (K - 1 - j)) & 1u) << op.tpos[j];
        off[m] = v;
    }
}

// Eq. 1 on one group: out[r] = sum_c G[r][c] a[c] for the touched rows.
template <typename R, int K>
__device__ __forceinline__ void dense_k(Cx<R>* s, uint32_t base, const uint32_t (&off)[1 << K], uint32_t touch,
                                        const Cx<R>* c) {
    Cx<R> a[1 << K];
#pragma unroll
    for (int m = 0; m < (1 << K); ++m) a[m] = s[base | off[m]];
#pragma unroll
    for (int row = 0; row < (1 << K); ++row) {
        if (!((touch >> row) & 1u)) continue;
        Cx<R> acc{R(0), R(0)};
#pragma unroll
        for (int col = 0; col < (1 << K); ++col) cfma(acc, c[row * (1 << K) + col], a[col]);
        s[base | off[row]] = acc;
    }
}

template <typename R, int K>
__device__ __forceinline__ void diag_k(Cx<R>* s, uint32_t base, const uint32_t (&off)[1 << K],
                                       const Cx<R>* c) {
#pragma unroll
    for (int m = 0; m < (1 << K); ++m) s[base | off[m]] = cmul(c[m], s[base | off[m]]);
}

template <typename R, int K>
__device__ __forceinline__ void run_op(Cx<R>* s, const SOp& op, uint32_t groups, const Cx<R>* c) {
    uint32_t off[1 << K];
    member_offsets<K>(op, off);
    for (uint32_t g = threadIdx.x; g < groups; g += kSmallThreads) {
        uint64_t b = g;
        for (int j = 0; j < op.nins; ++j) b = insert_zero(b, op.ins[j]);
        const uint32_t base = (uint32_t)b | (uint32_t)op.fval;
        if (op.kind == PK_DENSE) {
            dense_k<R, K>(s, base, off, op.touch, c);
        } else if (op.kind == PK_DIAG) {
            diag_k<R, K>(s, base, off, c);
        } else if constexpr (K == 1) {  // PK_X
            const Cx<R> a0 = s[base | off[0]], a1 = s[base | off[1]];
            s[base | off[0]] = a1;
            s[base | off[1]] = a0;
        } else if constexpr (K == 2) {  // PK_SWAP
            const Cx<R> a1 = s[base | off[1]], a2 = s[base | off[2]];
            s[base | off[1]] = a2;
            s[base | off[2]] = a1;
        } else if constexpr (K == 0) {  // PK_PHASE / PK_NEG
            const Cx<R> a = s[base];
            s[base] = op.kind == PK_NEG ? Cx<R>{-a.re, -a.im} : cmul(c[0], a);
        }
    }
}

// Program layout (device): CInfo[nchunks], then the chunks, each 16-byte
// aligned: SOp[nops] followed by the chunk's coefficients (op.data is
// relative to them).  Chunks are double-buffered into SMEM with cp.async, so
// every op reads its record and coefficients from shared memory.
struct CInfo {
    uint32_t off, bytes, nops, pad;
};
constexpr uint32_t kChunkBytes = 16384;

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void fetch_chunk(unsigned char* dst, const unsigned char* prog, const CInfo& ci) {
    for (uint32_t i = threadIdx.x * 16; i < ci.bytes; i += kSmallThreads * 16) cp16(dst + i, prog + ci.off + i);
    cp_commit();
}

template <typename R>
__global__ void __launch_bounds__(kSmallThreads) small_kernel(Cx<R>* psi, int n, const unsigned char* __restrict__ prog,
                                                              uint32_t nchunks) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx<R>* s = reinterpret_cast<Cx<R>*>(smem_raw);
    const uint32_t N = 1u << n;
    unsigned char* const buf0 = smem_raw + sizeof(Cx<R>) * N;  // chunk c lives at buf0 + (c & 1) * kChunkBytes
    const CInfo* info = reinterpret_cast<const CInfo*>(prog);
    if (nchunks > 0) fetch_chunk(buf0, prog, info[0]);
    for (uint32_t i = threadIdx.x; i < N; i += kSmallThreads) s[i] = psi[i];
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
        if (ch + 1 < nchunks) {
            fetch_chunk(buf0 + ((ch + 1) & 1) * kChunkBytes, prog, info[ch + 1]);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const uint32_t nops = info[ch].nops;
        unsigned char* const cb = buf0 + (ch & 1) * kChunkBytes;
        const SOp* ops = reinterpret_cast<const SOp*>(cb);
        const unsigned char* data = cb + nops * sizeof(SOp);  // op.data / DSub.coff are byte offsets
        for (uint32_t o = 0; o < nops; ++o) {
            const SOp& op = ops[o];  // read in place from SMEM (a local copy indexed dynamically spills)
            const uint32_t groups = N >> op.nins;
            const Cx<R>* c = reinterpret_cast<const Cx<R>*>(data + op.data);
            if (op.kind == PK_DRUN) {
                const DSub* sub = reinterpret_cast<const DSub*>(data + op.data);
                const int nsub = op.k;
                for (uint32_t i = threadIdx.x; i < N; i += kSmallThreads) {
                    Cx<R> a = s[i];
                    for (int j = 0; j < nsub; ++j) {
                        const DSub& d = sub[j];
                        if ((i & (uint32_t)d.fmask) != (uint32_t)d.fval) continue;
                        if (d.kind == PK_NEG) {
                            a = Cx<R>{-a.re, -a.im};
                            continue;
                        }
                        uint32_t row = 0;
                        for (int t = 0; t < d.k; ++t) row = (row << 1) | ((i >> d.tpos[t]) & 1u);
                        a = cmul(reinterpret_cast<const Cx<R>*>(data + d.coff)[row], a);
                    }
                    s[i] = a;
                }
                __syncthreads();
                continue;
            }
            switch (op.k) {
                case 0: run_op<R, 0>(s, op, groups, c); break;
                case 1: run_op<R, 1>(s, op, groups, c); break;
                case 2: run_op<R, 2>(s, op, groups, c); break;
                case 3: run_op<R, 3>(s, op, groups, c); break;
                default: run_op<R, 4>(s, op, groups, c); break;
            }
            __syncthreads();
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < N; i += kSmallThreads) psi[i] = s[i];
}

template <typename R>
std::vector<unsigned char> lower(const std::vector<Pass>& prog, uint32_t* nchunks_out) {
    struct Chunk {
        std::vector<SOp> ops;
        std::vector<unsigned char> data;  // 16-byte aligned records / coefficients
        size_t bytes() const { return ops.size() * sizeof(SOp) + data.size(); }
        uint32_t put(const void* p, size_t b) {
            const uint32_t at = (uint32_t)data.size();
            data.resize(at + ((b + 15) & ~size_t(15)), 0);
            if (b) std::memcpy(data.data() + at, p, b);
            return at;
        }
    };
    auto coeffs = [](const Pass& p) {
        std::vector<Cx<R>> v;
        for (const cd& z : p.m) v.push_back(Cx<R>{(R)z.real(), (R)z.imag()});
        return v;
    };
    auto is_diag = [](const Pass& p) {
        return p.kind == PK_PHASE || p.kind == PK_NEG || (p.kind == PK_DIAG && p.k <= 4);
    };
    auto padded = [](size_t b) { return (b + 15) & ~size_t(15); };
    std::vector<Chunk> chunks(1);
    for (size_t i = 0; i < prog.size();) {
        // a run of >= 2 consecutive diagonal passes -> one DRUN op
        size_t j = i;
        while (j < prog.size() && j - i < (size_t)kMaxRun && is_diag(prog[j])) ++j;
        if (j - i >= 2) {
            size_t need = sizeof(SOp) + padded((j - i) * sizeof(DSub));
            for (size_t q = i; q < j; ++q) need += padded(prog[q].m.size() * sizeof(Cx<R>));
            if (chunks.back().bytes() + need > kChunkBytes) chunks.emplace_back();
            Chunk& c = chunks.back();
            std::vector<DSub> subs(j - i);
            for (size_t q = i; q < j; ++q) {
                const Pass& p = prog[q];
                DSub& d = subs[q - i];
                std::memset(&d, 0, sizeof(d));
                d.kind = p.kind;
                d.k = p.kind == PK_DIAG ? p.k : 0;
                for (int t = 0; t < d.k; ++t) d.tpos[t] = (int8_t)p.tpos[t];
                for (int t = 0; t < p.nfix; ++t) {
                    d.fmask |= 1ull << p.fpos[t];
                    if (p.fval[t]) d.fval |= 1ull << p.fpos[t];
                }
                const std::vector<Cx<R>> v = coeffs(p);
                d.coff = v.empty() ? 0 : c.put(v.data(), v.size() * sizeof(Cx<R>));
            }
            SOp o;
            std::memset(&o, 0, sizeof(o));
            o.kind = PK_DRUN;
            o.k = (int32_t)(j - i);
            o.data = c.put(subs.data(), subs.size() * sizeof(DSub));
            c.ops.push_back(o);
            i = j;
            continue;
        }
        const Pass& p = prog[i++];
        SOp o;
        std::memset(&o, 0, sizeof(o));
        o.kind = p.kind;
        o.k = (p.kind == PK_PHASE || p.kind == PK_NEG) ? 0 : p.k;
        o.touch = p.touch;
        int ins[64], ni = 0;
        for (int t = 0; t < o.k; ++t) {
            o.tpos[t] = (int8_t)p.tpos[t];
            ins[ni++] = p.tpos[t];
        }
        for (int t = 0; t < p.nfix; ++t) {
            ins[ni++] = p.fpos[t];
            if (p.fval[t]) o.fval |= 1ull << p.fpos[t];
        }
        std::sort(ins, ins + ni);
        o.nins = ni;
        for (int t = 0; t < ni; ++t) o.ins[t] = (int8_t)ins[t];
        const std::vector<Cx<R>> v = coeffs(p);
        if (chunks.back().bytes() + sizeof(SOp) + padded(v.size() * sizeof(Cx<R>)) > kChunkBytes)
            chunks.emplace_back();
        Chunk& c = chunks.back();
        o.data = v.empty() ? 0 : c.put(v.data(), v.size() * sizeof(Cx<R>));
        c.ops.push_back(o);
    }
    if (chunks.back().ops.empty()) chunks.pop_back();
    const size_t head = ((chunks.size() * sizeof(CInfo)) + 15) & ~size_t(15);
    std::vector<CInfo> info(chunks.size());
    size_t off = head;
    for (size_t i = 0; i < chunks.size(); ++i) {
        const size_t b = (chunks[i].bytes() + 15) & ~size_t(15);
        info[i] = CInfo{(uint32_t)off, (uint32_t)b, (uint32_t)chunks[i].ops.size(), 0};
        off += b;
    }
    std::vector<unsigned char> blob(std::max<size_t>(off, 16), 0);
    if (!info.empty()) std::memcpy(blob.data(), info.data(), info.size() * sizeof(CInfo));
    for (size_t i = 0; i < chunks.size(); ++i) {
        unsigned char* d = blob.data() + info[i].off;
        std::memcpy(d, chunks[i].ops.data(), chunks[i].ops.size() * sizeof(SOp));
        if (!chunks[i].data.empty())
            std::memcpy(d + chunks[i].ops.size() * sizeof(SOp), chunks[i].data.data(), chunks[i].data.size());
    }
    *nchunks_out = (uint32_t)chunks.size();
    return blob;
}

template <typename R>
size_t smem_bytes(int nl) {
    return (sizeof(Cx<R>) << nl) + 2 * kChunkBytes;
}

template <typename R>
cudaError_t set_smem(int nl) {
    static int done_for = -1;
    const size_t smem = smem_bytes<R>(nl);
    if ((int)smem <= done_for) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(small_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)std::max<size_t>(smem, 48 * 1024));
    if (e == cudaSuccess) done_for = (int)std::max<size_t>(smem, 48 * 1024);
    return e;
}

template <typename R>
void launch(void* psi, int nl, const void* dev, uint32_t nchunks, cudaStream_t st) {
    small_kernel<R><<<1, kSmallThreads, smem_bytes<R>(nl), st>>>(static_cast<Cx<R>*>(psi), nl,
                                                               static_cast<const unsigned char*>(dev), nchunks);
}

}  // namespace

bool small_supports(const Pass& p) {
    switch (p.kind) {
        case PK_DENSE:
            return p.k <= kSmallMaxK;
        case PK_X:
        case PK_SWAP:
        case PK_PHASE:
        case PK_NEG:
            return true;
        case PK_DIAG:
            return p.k <= kSmallMaxK;
        default:
            return false;
    }
}

template <typename R>
cudaError_t small_prepare(const std::vector<Pass>& prog, void* psi, int nl, PreparedSmall& out) {
    uint32_t nchunks = 0;
    std::vector<unsigned char> blob = lower<R>(prog, &nchunks);
    cudaError_t e = set_smem<R>(nl);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&out.dev, blob.size());
    if (e != cudaSuccess) return e;
    e = cudaMemcpy(out.dev, blob.data(), blob.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return e;
    out.nchunks = nchunks;
    out.nl = nl;
    out.amp_bytes = (int)sizeof(Cx<R>);
    out.psi = psi;
    return cudaSuccess;
}

cudaError_t small_launch(const PreparedSmall& p, cudaStream_t st, LaunchStats& ls) {
    if (p.amp_bytes == 16) launch<double>(p.psi, p.nl, p.dev, p.nchunks, st);
    else launch<float>(p.psi, p.nl, p.dev, p.nchunks, st);
    ls.launches++;
    return cudaGetLastError();
}

void small_release(PreparedSmall& p) {
    if (p.dev) cudaFree(p.dev);
    p.dev = nullptr;
}

template <typename R>
cudaError_t run_small(const std::vector<Pass>& prog, void* psi, int nl, cudaStream_t st, LaunchStats& ls) {
    uint32_t nchunks = 0;
    std::vector<unsigned char> blob = lower<R>(prog, &nchunks);
    cudaError_t e = set_smem<R>(nl);
    if (e != cudaSuccess) return e;
    void* dev = nullptr;
    e = cudaMallocAsync(&dev, blob.size(), st);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(dev, blob.data(), blob.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
        // pageable source: the copy is staged before cudaMemcpyAsync returns, but
        // make the host buffer's lifetime independent of that detail
        e = cudaStreamSynchronize(st);
    }
    if (e == cudaSuccess) {
        launch<R>(psi, nl, dev, nchunks, st);
        ls.launches++;
        e = cudaGetLastError();
    }
    cudaFreeAsync(dev, st);
    return e;
}

template cudaError_t small_prepare<float>(const std::vector<Pass>&, void*, int, PreparedSmall&);
template cudaError_t small_prepare<double>(const std::vector<Pass>&, void*, int, PreparedSmall&);
template cudaError_t run_small<float>(const std::vector<Pass>&, void*, int, cudaStream_t, LaunchStats&);
template cudaError_t run_small<double>(const std::vector<Pass>&, void*, int, cudaStream_t, LaunchStats&);

}  // namespace qj
