// api.cu -- the C ABI of libqj (include/qj.h): validation, the per-gate
// planner (logical qubits -> physical bit positions, specialisation, sharded
// global-qubit handling) and dispatch to the sm_100a pass kernels.
//
// Nothing here does amplitude arithmetic: every amplitude is touched by a
// kernel in kernels.cuh / tile_pass.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "qj_internal.h"
#include "planner.h"
#include "common.cuh"
#include "dist.h"
#include "small.h"
#include "tile_jit.h"

using namespace qj;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;

static qj_status fail(qj_status code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

static qj_status cuda_fail(cudaError_t e, const char* where) {
    return fail(QJ_ERR_CUDA, "%s: %s (%s)", where, cudaGetErrorName(e), cudaGetErrorString(e));
}

// QJ_FUSE_GATES_K(k): fusion width in flag bits 4-7 (0 = the paper's 2)
static int fuse_width(uint32_t flags) {
    const int k = (int)((flags >> 4) & 15u);
    return k ? k : 2;
}

// ------------------------------------------------------------------ handle
struct qj_state_s {
    int n = 0, nl = 0, g = 0;
    qj_dtype dt = QJ_C128;
    int amp_bytes = 16;
    std::vector<void*> shards;
    cudaStream_t stream = nullptr;
    std::vector<int> phys;  // logical qubit -> physical bit (bits >= nl are global)
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    double* bins = nullptr;
    size_t bins_cap = 0;  // doubles
    LaunchStats ls;
    qj_counters ctr{};
    Planner planner;
    TileStaging stg;  // tile-pass program buffers
    // multi-GPU (NCCL): one shard per process, global shard index = rank
    void* comm = nullptr;  // ncclComm_t, nullptr for single-process states
    int rank = 0, nranks = 1;
    void* xbuf = nullptr;  // exchange staging ring
    size_t xbuf_bytes = 0;
    // exchange pipeline: NCCL transfers on their own stream, so chunk c's
    // transfer overlaps chunk c+1's pack and chunk c-1's unpack
    cudaStream_t xstream = nullptr;
    cudaEvent_t xev_in[2] = {}, xev_out[2] = {}, xev_start = nullptr;
    void* mbuf = nullptr;  // measurement scratch (norm partials, sampler CDF); never in a captured graph
    size_t mbuf_bytes = 0;
    // host-staged states (row f4): `shards` are HOST slices;
    // work streams them through three device buffers (H2D / compute / D2H on
    // separate streams).
    bool host = false;
    // half-slice table: logical slice r = halves[2r] (local top bit 0) and
    // halves[2r+1] (top bit 1), each 2^(nl-1) amplitudes of the caller's buffer.
    // Exchanges with the top local bit swap table entries (no data moves).
    std::vector<void*> halves;
    void* host_base = nullptr;
    struct HostPipe {
        bool ready = false;
        void* dbuf[3] = {};
        cudaStream_t h2d = nullptr, d2h = nullptr;
        cudaEvent_t up[3] = {}, done[3] = {}, freed[3] = {}, mark = nullptr, tail = nullptr;
    } hp;
    int total_shards() const { return comm ? nranks : (int)shards.size(); }
    // circuits seen before: plan + prepared tile passes (+ a CUDA graph)
    struct CachedPlan {
        std::vector<uint64_t> key;
        std::vector<Step> steps;
        std::vector<int> phys_after;
        std::vector<PreparedTile> tiles;  // one per TILE step, in order
        std::vector<PreparedSmall> smalls;  // one per SMALL step, in order
        // qj_simulate plans: |basis> synthesised by the first tile pass (else an
        // init launch), the marginal fused into the last tile pass (else a
        // marginal launch), bins owned by the plan
        bool sim = false, init_first = false, marg_last = false, init_none = false;
        uint64_t basis = 0;
        int nq = 0;
        int qpos[16] = {};
        double* sim_bins = nullptr;
        void* out = nullptr;
        cudaGraphExec_t exec = nullptr;
        bool graphable = true;
        uint64_t uses = 0, kernels = 0;
    };
    std::vector<CachedPlan*> plans;  // most recent first
    bool cache_on = true;
    // profiling: event pairs around passes
    bool profiling = false;
    struct Rec {
        int kind;
        double bytes;
        cudaEvent_t a, b;
    };
    std::vector<Rec> recs;
    std::vector<cudaEvent_t> pool;
};

static const char* kProfNames[] = {"gate_dense", "gate_x",     "gate_swap", "diag_table", "diag_phase",
                                   "diag_neg",   "tile",       "exchange",  "small",     "init"};
enum { PROF_TILE = 6, PROF_EXCHANGE = 7, PROF_SMALL = 8, PROF_INIT = 9, PROF_N = 10 };

namespace {

bool dtype_ok(int dt) { return dt == QJ_C64 || dt == QJ_C128; }

template <typename F>
cudaError_t by_dtype(qj_dtype dt, F&& f) {
    if (dt == QJ_C64) return f((float)0);
    return f((double)0);
}

qj_status ensure_scratch(qj_state s, size_t bytes) {
    if (s->scratch_bytes >= bytes) return QJ_OK;
    if (s->scratch) {
        cudaStreamSynchronize(s->stream);
        cudaFree(s->scratch);
        s->scratch = nullptr;
        s->scratch_bytes = 0;
    }
    cudaError_t e = cudaMalloc(&s->scratch, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "scratch alloc");
    s->scratch_bytes = bytes;
    return QJ_OK;
}

qj_status ensure_mbuf(qj_state s, size_t bytes) {
    if (s->mbuf_bytes >= bytes) return QJ_OK;
    if (s->mbuf) {
        cudaStreamSynchronize(s->stream);
        cudaFree(s->mbuf);
        s->mbuf = nullptr;
        s->mbuf_bytes = 0;
    }
    cudaError_t e = cudaMalloc(&s->mbuf, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "measurement scratch alloc");
    s->mbuf_bytes = bytes;
    return QJ_OK;
}

qj_status ensure_bins(qj_state s, size_t nb) {
    if (s->bins_cap >= nb) return QJ_OK;
    if (s->bins) {
        cudaStreamSynchronize(s->stream);
        cudaFree(s->bins);
        s->bins = nullptr;
        s->bins_cap = 0;
    }
    cudaError_t e = cudaMalloc(&s->bins, nb * sizeof(double));
    if (e != cudaSuccess) return cuda_fail(e, "bins alloc");
    s->bins_cap = nb;
    return QJ_OK;
}

// Read a host complex array of the state's dtype into complex<double>.
std::vector<cd> read_complex(const void* p, size_t count, qj_dtype dt) {
    std::vector<cd> v(count);
    if (dt == QJ_C64) {
        const float* f = static_cast<const float*>(p);
        for (size_t i = 0; i < count; ++i) v[i] = cd(f[2 * i], f[2 * i + 1]);
    } else {
        const double* d = static_cast<const double*>(p);
        for (size_t i = 0; i < count; ++i) v[i] = cd(d[2 * i], d[2 * i + 1]);
    }
    return v;
}

qj_status validate_qubits(qj_state s, const int* targets, int nt, const int* controls, int nc) {
    if (nt < 1) return fail(QJ_ERR_INVALID_ARG, "nt must be >= 1 (got %d)", nt);
    if (nt > QJ_MAX_TARGETS) return fail(QJ_ERR_TOO_MANY_TARGETS, "nt=%d exceeds %d", nt, QJ_MAX_TARGETS);
    if (nc < 0) return fail(QJ_ERR_INVALID_ARG, "nc must be >= 0 (got %d)", nc);
    if (nc > QJ_MAX_CONTROLS) return fail(QJ_ERR_TOO_MANY_TARGETS, "nc=%d exceeds %d", nc, QJ_MAX_CONTROLS);
    if (!targets) return fail(QJ_ERR_INVALID_ARG, "targets is NULL");
    if (nc > 0 && !controls) return fail(QJ_ERR_INVALID_ARG, "controls is NULL with nc=%d", nc);
    uint64_t seen_lo = 0, seen_hi = 0;
    auto check = [&](int q, const char* what) -> qj_status {
        if (q < 0 || q >= s->n) return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "%s qubit %d out of range [0,%d)", what, q, s->n);
        uint64_t& w = q < 64 ? seen_lo : seen_hi;
        const uint64_t b = 1ull << (q & 63);
        if (w & b) return fail(QJ_ERR_OVERLAPPING_QUBITS, "qubit %d listed twice (targets and controls must be disjoint)", q);
        w |= b;
        return QJ_OK;
    };
    for (int i = 0; i < nt; ++i)
        if (qj_status st = check(targets[i], "target")) return st;
    for (int i = 0; i < nc; ++i)
        if (qj_status st = check(controls[i], "control")) return st;
    return QJ_OK;
}

// Convert an ABI gate into a logical gate (validated).
qj_status make_lgate(qj_state s, int kind, const int* targets, int nt, const int* controls, int nc,
                     const void* data, LGate& out) {
    if (qj_status st = validate_qubits(s, targets, nt, controls, nc)) return st;
    out = LGate();
    out.kind = kind;
    out.nt = nt;
    out.nc = nc;
    for (int i = 0; i < nt; ++i) out.t[i] = targets[i];
    for (int i = 0; i < nc; ++i) out.c[i] = controls[i];
    switch (kind) {
        case QJ_GATE_DENSE:
            if (!data) return fail(QJ_ERR_INVALID_ARG, "matrix is NULL");
            out.data = read_complex(data, (size_t)1 << (2 * nt), s->dt);
            break;
        case QJ_GATE_X:
        case QJ_GATE_Z:
            if (nt != 1) return fail(QJ_ERR_INVALID_ARG, "X/Z take exactly one target (got %d)", nt);
            break;
        case QJ_GATE_SWAP:
            if (nt != 2) return fail(QJ_ERR_INVALID_ARG, "SWAP takes exactly two targets (got %d)", nt);
            break;
        case QJ_GATE_FSIM:
            if (nt != 2) return fail(QJ_ERR_INVALID_ARG, "fSim takes exactly two targets (got %d)", nt);
            if (!data) return fail(QJ_ERR_INVALID_ARG, "fSim parameters are NULL");
            out.data = read_complex(data, 5, s->dt);
            break;
        case QJ_GATE_DIAG:
            if (!data) return fail(QJ_ERR_INVALID_ARG, "diagonal is NULL");
            out.data = read_complex(data, (size_t)1 << nt, s->dt);
            break;
        default:
            return fail(QJ_ERR_INVALID_ARG, "unknown gate kind %d", kind);
    }
    return QJ_OK;
}

cudaEvent_t pool_get(qj_state s) {
    if (!s->pool.empty()) {
        cudaEvent_t e = s->pool.back();
        s->pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    qj_state s;
    int kind;
    double bytes;
    cudaEvent_t a = nullptr;
    ProfScope(qj_state s_, int kind_, double bytes_) : s(s_), kind(kind_), bytes(bytes_) {
        if (!s->profiling) return;
        a = pool_get(s);
        cudaEventRecord(a, s->stream);
    }
    ~ProfScope() {
        if (!a) return;
        cudaEvent_t b = pool_get(s);
        cudaEventRecord(b, s->stream);
        s->recs.push_back({kind, bytes, a, b});
    }
};

int prof_kind(const Step& st) {
    if (st.type == Step::TILE) return PROF_TILE;
    if (st.type == Step::SMALL) return PROF_SMALL;
    return st.pass.kind;
}

// Execute planned steps on the device.
// Exchange over NCCL (dist.h): this rank trades the half of its shard whose
// local bit L equals spec.half_bit with the partner, chunk by chunk through
// the staging ring.
qj_status nccl_exchange_with(qj_state s, const ExchangeSpec& ex, int L);

qj_status nccl_exchange(qj_state s, int j, int L) { return nccl_exchange_with(s, exchange_spec(s->rank, j), L); }

// The exchange proper (also driven directly by qj_debug_nccl_self_exchange).
qj_status nccl_exchange_with(qj_state s, const ExchangeSpec& ex, int L) {
    const char* why = nullptr;
    const NcclApi* api = nccl_api(&why);
    if (!api) return fail(QJ_ERR_NCCL, "NCCL unavailable: %s", why ? why : "?");
    const uint64_t half = 1ull << (s->nl - 1);
    const uint64_t chunk = std::min<uint64_t>(half, (uint64_t)(256ull << 20) / (uint64_t)s->amp_bytes);
    const bool contiguous = (L == s->nl - 1);
    const size_t cb = (size_t)chunk * s->amp_bytes;
    const size_t need = contiguous ? 2 * cb : 4 * cb;  // 2 receive slots (+ 2 pack slots)
    if (s->xbuf_bytes < need) {
        if (s->xbuf) {
            cudaStreamSynchronize(s->stream);
            cudaFree(s->xbuf);
            s->xbuf = nullptr;
            s->xbuf_bytes = 0;
        }
        cudaError_t e = cudaMalloc(&s->xbuf, need);
        if (e != cudaSuccess) return cuda_fail(e, "exchange staging alloc");
        s->xbuf_bytes = need;
    }
    if (!s->xstream) {
        cudaError_t e = cudaStreamCreateWithFlags(&s->xstream, cudaStreamNonBlocking);
        for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
            e = cudaEventCreateWithFlags(&s->xev_in[k], cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->xev_out[k], cudaEventDisableTiming);
        }
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s->xev_start, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "exchange stream");
    }
    unsigned char* state = static_cast<unsigned char*>(s->shards[0]);
    unsigned char* stage = static_cast<unsigned char*>(s->xbuf);
    ncclComm_t comm = static_cast<ncclComm_t>(s->comm);
    const uint64_t base = (uint64_t)ex.half_bit << (s->nl - 1);  // contiguous case
    // Pipeline over chunks, two staging slots:
    //   compute stream: [pack c -> slot c&1] ... [unpack slot c&1 -> state]
    //   exchange stream:        [send c / recv c into slot c&1]
    // xev_in[k]:  slot k's send data is ready (pack done, or the state itself
    //             is ready) and its receive buffer is free (unpack c-2 done);
    // xev_out[k]: chunk c's transfer finished (the unpack may read slot k and
    //             overwrite the amplitudes it sent).
    // The compute stream waits for the last transfer before its last unpack,
    // so both streams join there (also inside a captured CUDA graph).
    cudaError_t e = cudaEventRecord(s->xev_start, s->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s->xstream, s->xev_start, 0);
    if (e != cudaSuccess) return cuda_fail(e, "exchange fork");
    for (uint64_t h0 = 0, c = 0; h0 < half; h0 += chunk, ++c) {
        const int k = (int)(c & 1);
        const uint64_t cnt = std::min<uint64_t>(chunk, half - h0);
        const size_t bytes = (size_t)cnt * s->amp_bytes;
        unsigned char* recv = stage + k * cb;
        const unsigned char* send;
        if (contiguous) {
            send = state + (size_t)(base + h0) * s->amp_bytes;
        } else {
            unsigned char* pk = stage + (2 + k) * cb;
            e = launch_half_pack(state, pk, s->amp_bytes, L, ex.half_bit, h0, cnt, s->stream);
            if (e != cudaSuccess) return cuda_fail(e, "exchange pack");
            s->ls.launches++;
            send = pk;
        }
        e = cudaEventRecord(s->xev_in[k], s->stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s->xstream, s->xev_in[k], 0);
        if (e != cudaSuccess) return cuda_fail(e, "exchange order");
        ncclResult_t r = api->GroupStart();
        if (r == ncclSuccess) r = api->Send(send, bytes, ncclInt8, ex.peer, comm, s->xstream);
        if (r == ncclSuccess) r = api->Recv(recv, bytes, ncclInt8, ex.peer, comm, s->xstream);
        const ncclResult_t r2 = api->GroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(QJ_ERR_NCCL, "exchange send/recv with rank %d: %s", ex.peer,
                        api->GetErrorString(r != ncclSuccess ? r : r2));
        e = cudaEventRecord(s->xev_out[k], s->xstream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, s->xev_out[k], 0);
        if (e != cudaSuccess) return cuda_fail(e, "exchange order");
        if (contiguous) e = launch_copy(state + (size_t)(base + h0) * s->amp_bytes, recv, bytes, s->stream);
        else e = launch_half_unpack(state, recv, s->amp_bytes, L, ex.half_bit, h0, cnt, s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "exchange unpack");
        s->ls.launches++;
    }
    return QJ_OK;
}

// Device pointer of global shard `g` if this process owns it, else nullptr.
void* shard_ptr(qj_state s, int g) {
    if (s->comm) return g == s->rank ? s->shards[0] : nullptr;
    return s->shards[(size_t)g];
}

// ---- host-staged execution -------------------------------------------------
void host_identity_halves(qj_state s) {
    const size_t hb = ((size_t)s->amp_bytes << s->nl) / 2;
    s->halves.resize(2 * s->shards.size());
    for (size_t h = 0; h < s->halves.size(); ++h) s->halves[h] = static_cast<unsigned char*>(s->host_base) + h * hb;
}

void copy_par(void* dst, const void* src, size_t bytes) {
    const size_t kMin = 64ull << 20;
    const unsigned nt = bytes < kMin ? 1u : std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
    if (nt == 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    const size_t per = (bytes + nt - 1) / nt;
    for (unsigned t = 0; t < nt; ++t) {
        const size_t b = t * per, e = std::min(bytes, b + per);
        if (b >= e) break;
        th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + b, static_cast<const char*>(src) + b, e - b); });
    }
    for (auto& x : th) x.join();
}

// Move the half-slices back to their canonical places in the caller's buffer
// (cycle by cycle through one temporary half).  The stream must be idle.
qj_status host_materialize(qj_state s) {
    const size_t nh = s->halves.size();
    const size_t hb = ((size_t)s->amp_bytes << s->nl) / 2;
    auto home = [&](size_t h) { return static_cast<unsigned char*>(s->host_base) + h * hb; };
    // where[h] = index of the home block currently holding logical half h's data
    std::vector<size_t> where(nh);
    for (size_t h = 0; h < nh; ++h) where[h] = (size_t)(static_cast<unsigned char*>(s->halves[h]) -
                                                         static_cast<unsigned char*>(s->host_base)) / hb;
    bool identity = true;
    for (size_t h = 0; h < nh; ++h) identity &= where[h] == h;
    if (identity) return QJ_OK;
    std::vector<unsigned char> tmp;
    try {
        tmp.resize(hb);
    } catch (...) {
        return fail(QJ_ERR_CAPACITY, "host materialise: no memory for a %zu-byte temporary", hb);
    }
    std::vector<char> done(nh, 0);
    for (size_t h = 0; h < nh; ++h) {
        if (done[h] || where[h] == h) {
            done[h] = 1;
            continue;
        }
        // cycle: home(h) must receive block where[h]; save home(h) first
        copy_par(tmp.data(), home(h), hb);
        size_t cur = h;
        // the block originally at home(h) belongs to logical half k with where[k] == h
        while (true) {
            const size_t src = where[cur];
            done[cur] = 1;
            if (src == h) {
                copy_par(home(cur), tmp.data(), hb);
                break;
            }
            copy_par(home(cur), home(src), hb);
            cur = src;
            // the data now needed at home(src) is logical half `src`'s, stored at where[src]
        }
    }
    host_identity_halves(s);
    return QJ_OK;
}

qj_status host_pipe_init(qj_state s) {
    auto& p = s->hp;
    if (p.ready) return QJ_OK;
    const size_t bytes = (size_t)s->amp_bytes << s->nl;
    cudaError_t e = cudaSuccess;
    for (int b = 0; b < 3 && e == cudaSuccess; ++b) e = cudaMalloc(&p.dbuf[b], bytes);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking);
    for (int b = 0; b < 3 && e == cudaSuccess; ++b) {
        e = cudaEventCreateWithFlags(&p.up[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.done[b], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.freed[b], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.mark, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.tail, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_fail(e, "host-staging pipeline setup (3 slice buffers)");
    p.ready = true;
    return QJ_OK;
}

// Stream the listed host slices through the device: slice t is uploaded on the
// H2D stream into buffer t mod 3, `compute(r, dev_ptr)` is enqueued on the
// handle's stream, and (write_back) the buffer is copied back on the D2H
// stream, so upload, compute and download of consecutive slices overlap.  The
// handle's stream waits for the last write-back, so anything enqueued on it
// afterwards (and qj_sync) sees the updated host slices.
template <typename F>
qj_status host_sweep(qj_state s, const std::vector<int>& slices, bool write_back, F&& compute) {
    if (slices.empty()) return QJ_OK;
    if (qj_status q = host_pipe_init(s)) return q;
    auto& p = s->hp;
    const size_t bytes = (size_t)s->amp_bytes << s->nl;
    cudaError_t e = cudaEventRecord(p.mark, s->stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p.h2d, p.mark, 0);
    bool used[3] = {false, false, false};
    for (size_t t = 0; t < slices.size() && e == cudaSuccess; ++t) {
        const int b = (int)(t % 3);
        const int r = slices[t];
        if (used[b]) e = cudaStreamWaitEvent(p.h2d, p.freed[b], 0);
        const size_t hb = bytes / 2;
        unsigned char* db = static_cast<unsigned char*>(p.dbuf[b]);
        if (e == cudaSuccess) e = cudaMemcpyAsync(db, s->halves[2 * (size_t)r], hb, cudaMemcpyHostToDevice, p.h2d);
        if (e == cudaSuccess) e = cudaMemcpyAsync(db + hb, s->halves[2 * (size_t)r + 1], hb, cudaMemcpyHostToDevice, p.h2d);
        if (e == cudaSuccess) e = cudaEventRecord(p.up[b], p.h2d);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, p.up[b], 0);
        if (e == cudaSuccess) e = compute(r, p.dbuf[b]);
        if (e != cudaSuccess) break;
        if (write_back) {
            e = cudaEventRecord(p.done[b], s->stream);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(p.d2h, p.done[b], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(s->halves[2 * (size_t)r], db, hb, cudaMemcpyDeviceToHost, p.d2h);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(s->halves[2 * (size_t)r + 1], db + hb, hb, cudaMemcpyDeviceToHost, p.d2h);
            if (e == cudaSuccess) e = cudaEventRecord(p.freed[b], p.d2h);
        } else {
            e = cudaEventRecord(p.freed[b], s->stream);
        }
        used[b] = true;
    }
    if (e == cudaSuccess && write_back) {
        e = cudaEventRecord(p.tail, p.d2h);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s->stream, p.tail, 0);
    }
    if (e != cudaSuccess) return cuda_fail(e, "host-staged sweep");
    return QJ_OK;
}

qj_status run_step_on(qj_state s, const Step& st, void* ptr) {
    if (st.type == Step::PASS && st.pass.k > 5 && st.pass.kind == PK_DENSE) {
        const size_t need = (size_t)s->amp_bytes * ((size_t)1 << (2 * st.pass.k));
        if (qj_status q = ensure_scratch(s, need)) return q;
    }
    ProfScope prof(s, prof_kind(st), st.alg_bytes);
    cudaError_t e = by_dtype(s->dt, [&](auto z) {
        using R = decltype(z);
        if (st.type == Step::TILE) return run_tile<R>(st.tile, ptr, s->nl, s->stream, s->stg, s->ls);
        if (st.type == Step::SMALL) return run_small<R>(st.prog, ptr, s->nl, s->stream, s->ls);
        return run_pass<R>(st.pass, ptr, s->nl, s->stream, s->scratch, s->scratch_bytes, s->ls);
    });
    if (e != cudaSuccess) return cuda_fail(e, "pass launch");
    s->ctr.passes++;
    s->ctr.alg_bytes += st.alg_bytes;
    return QJ_OK;
}

// Runs of per-slice steps between exchanges execute as ONE sweep over the
// slices (each slice uploaded once, all its steps applied, written back once).
// An exchange uploads each slice pair, swaps the halves in HBM and writes both
// back.  Bit for bit the same kernels as the in-HBM sharded path.
qj_status execute_host(qj_state s, const std::vector<Step>& steps_in) {
    const size_t nsh = s->shards.size();
    // exchanges with a lower local bit L: SWAP(L, top) on every slice, the
    // zero-copy exchange with the top bit, SWAP(L, top) again (the SWAP passes
    // join the neighbouring sweeps)
    std::vector<Step> steps;
    for (const Step& st : steps_in) {
        if (st.type != Step::EXCHANGE || st.lbit == s->nl - 1) {
            steps.push_back(st);
            continue;
        }
        auto swaps = [&]() {
            for (size_t r = 0; r < nsh; ++r) {
                Step w;
                w.type = Step::PASS;
                w.shard = (int)r;
                w.pass.kind = PK_SWAP;
                w.pass.k = 2;
                w.pass.tpos[0] = st.lbit;
                w.pass.tpos[1] = s->nl - 1;
                w.alg_bytes = pass_alg_bytes(w.pass, s->nl, s->amp_bytes);
                steps.push_back(std::move(w));
            }
        };
        swaps();
        Step x = st;
        x.lbit = s->nl - 1;
        steps.push_back(x);
        swaps();
    }
    size_t i = 0;
    while (i < steps.size()) {
        if (steps[i].type == Step::EXCHANGE) {
            // global bit j <-> top local bit: relabel half-slices (zero copy)
            const Step& st = steps[i++];
            for (size_t r = 0; r < nsh; ++r) {
                if ((r >> st.gbit) & 1) continue;
                const size_t r2 = r | (1ull << st.gbit);
                std::swap(s->halves[2 * r + 1], s->halves[2 * r2]);
            }
            s->ctr.exchanges++;
            continue;
        }
        size_t j = i;
        while (j < steps.size() && steps[j].type != Step::EXCHANGE) ++j;
        std::vector<std::vector<size_t>> per(nsh);
        for (size_t k = i; k < j; ++k)
            if (steps[k].shard >= 0 && (size_t)steps[k].shard < nsh) per[(size_t)steps[k].shard].push_back(k);
        std::vector<int> slices;
        for (size_t r = 0; r < nsh; ++r)
            if (!per[r].empty()) slices.push_back((int)r);
        qj_status inner = QJ_OK;
        qj_status q = host_sweep(s, slices, true, [&](int r, void* dptr) -> cudaError_t {
            for (size_t k : per[(size_t)r])
                if ((inner = run_step_on(s, steps[k], dptr)) != QJ_OK) return cudaErrorUnknown;
            return cudaSuccess;
        });
        if (inner != QJ_OK) return inner;
        if (q != QJ_OK) return q;
        i = j;
    }
    s->ctr.launches = s->ls.launches;
    return QJ_OK;
}

qj_status execute(qj_state s, const std::vector<Step>& steps) {
    if (s->host) return execute_host(s, steps);
    cudaError_t e = cudaSuccess;
    for (const Step& st : steps) {
        if (st.type == Step::EXCHANGE) {
            const double xb = (double)s->amp_bytes * (double)(1ull << (s->nl - 1)) * (double)s->shards.size();
            ProfScope prof(s, PROF_EXCHANGE, xb);
            // swap global bit (nl + j) with local bit L: pair shards r (bit j = 0) and r | 1<<j
            const int j = st.gbit, L = st.lbit;
            if (s->comm) {
                if (qj_status q = nccl_exchange(s, j, L)) return q;
                s->ctr.exchanges++;
                s->ctr.exchange_bytes += xb;
                continue;
            }
            for (size_t r = 0; r < s->shards.size(); ++r) {
                if ((r >> j) & 1) continue;
                const size_t r2 = r | (1ull << j);
                e = by_dtype(s->dt, [&](auto z) {
                    using R = decltype(z);
                    return run_exchange<R>(s->shards[r], s->shards[r2], s->nl, L, s->stream, s->ls);
                });
                if (e != cudaSuccess) return cuda_fail(e, "exchange launch");
            }
            s->ctr.exchanges++;
            s->ctr.exchange_bytes += xb;
            continue;
        }
        if (st.pass.k > 5 && st.pass.kind == PK_DENSE) {
            const size_t need = (size_t)s->amp_bytes * ((size_t)1 << (2 * st.pass.k));
            if (qj_status q = ensure_scratch(s, need)) return q;
        }
        void* ptr = shard_ptr(s, st.shard);
        if (!ptr) continue;  // another rank's shard
        ProfScope prof(s, prof_kind(st), st.alg_bytes);
        e = by_dtype(s->dt, [&](auto z) {
            using R = decltype(z);
            if (st.type == Step::TILE) return run_tile<R>(st.tile, ptr, s->nl, s->stream, s->stg, s->ls);
            if (st.type == Step::SMALL) return run_small<R>(st.prog, ptr, s->nl, s->stream, s->ls);
            return run_pass<R>(st.pass, ptr, s->nl, s->stream, s->scratch, s->scratch_bytes, s->ls);
        });
        if (e != cudaSuccess) return cuda_fail(e, "pass launch");
        s->ctr.passes++;
        s->ctr.alg_bytes += st.alg_bytes;
    }
    s->ctr.launches = s->ls.launches;
    return QJ_OK;
}

qj_status apply_lgates(qj_state s, const std::vector<LGate>& gates, bool fuse) {
    std::vector<Step> steps;
    PlanContext ctx{s->n, s->nl, s->g, s->amp_bytes, s->total_shards(), &s->phys};
    s->planner.plan(ctx, gates, fuse, steps);
    return execute(s, steps);
}

// ---- plan cache ---------------------------------------------------------
// The key is the exact request: flags, the qubit map at entry and every gate
// (kind, qubits, data bit patterns).  A hit skips planning, lowering and the
// tile program uploads; from the second use on the launches are replayed as a
// CUDA graph (one launch per circuit).
std::vector<uint64_t> plan_key(qj_state s, const qj_gate* gates, int ngates, uint32_t flags) {
    std::vector<uint64_t> k;
    k.reserve(8 + (size_t)ngates * 12);
    k.push_back(flags);
    k.push_back((uint64_t)s->n);
    for (int q = 0; q < s->n; ++q) k.push_back((uint64_t)s->phys[q]);
    k.push_back((uint64_t)ngates);
    for (int i = 0; i < ngates; ++i) {
        const qj_gate& g = gates[i];
        k.push_back(((uint64_t)g.kind << 40) | ((uint64_t)g.nt << 20) | (uint64_t)g.nc);
        uint64_t w = 0;
        for (int j = 0; j < g.nt; ++j) w = (w << 6) | (uint64_t)g.targets[j];
        k.push_back(w);
        w = 0;
        for (int j = 0; j < g.nc; ++j) w = (w << 6) | (uint64_t)g.controls[j];
        k.push_back(w);
        size_t cnt = 0;
        if (g.kind == QJ_GATE_DENSE) cnt = (size_t)1 << (2 * g.nt);
        else if (g.kind == QJ_GATE_DIAG) cnt = (size_t)1 << g.nt;
        else if (g.kind == QJ_GATE_FSIM) cnt = 5;
        const size_t words = cnt * (size_t)s->amp_bytes / 8;
        const uint64_t* p = static_cast<const uint64_t*>(g.data);
        for (size_t j = 0; j < words; ++j) {
            uint64_t v;
            std::memcpy(&v, p + j, 8);
            k.push_back(v);
        }
    }
    return k;
}

void release_plan(qj_state_s::CachedPlan* p) {
    if (p->exec) cudaGraphExecDestroy(p->exec);
    for (auto& t : p->tiles) tile_release(t);
    for (auto& t : p->smalls) small_release(t);
    if (p->sim_bins) cudaFree(p->sim_bins);
    delete p;
}

qj_status run_cached(qj_state s, qj_state_s::CachedPlan& p) {
    cudaError_t e = cudaSuccess;
    size_t ti = 0, si = 0;
    for (const Step& st : p.steps) {
        if (st.type == Step::EXCHANGE) {
            for (size_t r = 0; r < s->shards.size(); ++r) {
                if ((r >> st.gbit) & 1) continue;
                const size_t r2 = r | (1ull << st.gbit);
                e = by_dtype(s->dt, [&](auto z) {
                    using R = decltype(z);
                    return run_exchange<R>(s->shards[r], s->shards[r2], s->nl, st.lbit, s->stream, s->ls);
                });
                if (e != cudaSuccess) return cuda_fail(e, "exchange launch");
            }
            continue;
        }
        ProfScope prof(s, prof_kind(st), st.alg_bytes);
        if (st.type == Step::TILE) {
            e = tile_launch_prepared(p.tiles[ti++], s->stream, s->ls);
        } else if (st.type == Step::SMALL) {
            e = small_launch(p.smalls[si++], s->stream, s->ls);
        } else {
            void* ptr = shard_ptr(s, st.shard);
            e = by_dtype(s->dt, [&](auto z) {
                using R = decltype(z);
                return run_pass<R>(st.pass, ptr, s->nl, s->stream, s->scratch, s->scratch_bytes, s->ls);
            });
        }
        if (e != cudaSuccess) return cuda_fail(e, "cached pass launch");
    }
    return QJ_OK;
}

void account(qj_state s, const qj_state_s::CachedPlan& p) {
    for (const Step& st : p.steps) {
        if (st.type == Step::EXCHANGE) {
            s->ctr.exchanges++;
            s->ctr.exchange_bytes += (double)s->amp_bytes * (double)(1ull << (s->nl - 1)) * (double)s->shards.size();
        } else {
            s->ctr.passes++;
            s->ctr.alg_bytes += st.alg_bytes;
        }
    }
}

// Returns QJ_OK with *done = false when the request is not cacheable.
qj_status apply_circuit_cached(qj_state s, const qj_gate* gates, int ngates, uint32_t flags,
                               const std::vector<LGate>& gs, bool* done) {
    *done = false;
    if (!s->cache_on || s->comm || s->host) return QJ_OK;
    std::vector<uint64_t> key = plan_key(s, gates, ngates, flags);
    for (size_t i = 0; i < s->plans.size(); ++i) {
        qj_state_s::CachedPlan* p = s->plans[i];
        if (p->key != key) continue;
        std::rotate(s->plans.begin(), s->plans.begin() + (long)i, s->plans.begin() + (long)i + 1);
        const uint64_t before = s->ls.launches;
        const bool graph_ok = p->graphable && !s->profiling && s->stream != nullptr;
        if (graph_ok && !p->exec && p->uses >= 1) {
            cudaGraph_t g = nullptr;
            cudaError_t e = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) return cuda_fail(e, "graph capture");
            qj_status q = run_cached(s, *p);
            e = cudaStreamEndCapture(s->stream, &g);
            if (q != QJ_OK) return q;
            if (e != cudaSuccess) return cuda_fail(e, "graph capture end");
            e = cudaGraphInstantiate(&p->exec, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) {
                p->exec = nullptr;
                p->graphable = false;
                cudaGetLastError();
                return cuda_fail(e, "graph instantiate");
            }
            s->ls.launches = before;  // captured, not run
        }
        if (graph_ok && p->exec) {
            cudaError_t e = cudaGraphLaunch(p->exec, s->stream);
            if (e != cudaSuccess) return cuda_fail(e, "graph launch");
            s->ls.launches += p->kernels;
        } else {
            if (qj_status q = run_cached(s, *p)) return q;
        }
        p->uses++;
        account(s, *p);
        s->phys = p->phys_after;
        s->ctr.launches = s->ls.launches;
        *done = true;
        return QJ_OK;
    }
    // miss: plan, prepare the tile passes, run, remember
    auto* p = new qj_state_s::CachedPlan;
    p->key.swap(key);
    PlanContext ctx{s->n, s->nl, s->g, s->amp_bytes, s->total_shards(), &s->phys};
    s->planner.auto_fuse_ = !(flags & QJ_FUSE_GATES);
    s->planner.plan(ctx, gs, (flags & QJ_FUSE) != 0, p->steps);
    for (const Step& st : p->steps) {
        if (st.type == Step::TILE) {
            PreparedTile t;
            cudaError_t e = by_dtype(s->dt, [&](auto z) {
                using R = decltype(z);
                return tile_prepare<R>(st.tile, shard_ptr(s, st.shard), s->nl, t);
            });
            if (e != cudaSuccess) {
                release_plan(p);
                return cuda_fail(e, "tile prepare");
            }
            p->tiles.push_back(std::move(t));
        } else if (st.type == Step::SMALL) {
            PreparedSmall t;
            cudaError_t e = by_dtype(s->dt, [&](auto z) {
                using R = decltype(z);
                return small_prepare<R>(st.prog, shard_ptr(s, st.shard), s->nl, t);
            });
            if (e != cudaSuccess) {
                small_release(t);
                release_plan(p);
                return cuda_fail(e, "small prepare");
            }
            p->smalls.push_back(t);
        } else if (st.type == Step::PASS && st.pass.k > 5 && st.pass.kind == PK_DENSE) {
            p->graphable = false;  // big-k passes stage their matrix with a host copy
            const size_t need = (size_t)s->amp_bytes * ((size_t)1 << (2 * st.pass.k));
            if (qj_status q = ensure_scratch(s, need)) {
                release_plan(p);
                return q;
            }
        }
    }
    p->phys_after = s->phys;
    const uint64_t before = s->ls.launches;
    if (qj_status q = run_cached(s, *p)) {
        release_plan(p);
        return q;
    }
    p->kernels = s->ls.launches - before;
    p->uses = 1;
    account(s, *p);
    s->ctr.launches = s->ls.launches;
    s->plans.insert(s->plans.begin(), p);
    if (s->plans.size() > 16) {
        release_plan(s->plans.back());
        s->plans.pop_back();
    }
    *done = true;
    return QJ_OK;
}

}  // namespace

// ===================================================================== ABI
extern "C" {

const char* qj_last_error(void) { return g_err.c_str(); }

const char* qj_version(void) { return "qj 0.1 (sm_100a)"; }

uint64_t qj_insert_zero_bits(uint64_t g, const int* sorted_pos, int npos) {
    for (int i = 0; i < npos; ++i) g = insert_zero(g, sorted_pos[i]);
    return g;
}

static qj_status init_common(qj_state* out, void* const* shards, int nshards, int n, qj_dtype dt,
                             uint64_t basis_index, void* cuda_stream, void* comm = nullptr, int rank = 0,
                             int nranks = 1, bool host = false) {
    if (!out) return fail(QJ_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    if (!dtype_ok(dt)) return fail(QJ_ERR_DTYPE, "unknown dtype %d", (int)dt);
    if (n < 1 || n > QJ_MAX_QUBITS) return fail(QJ_ERR_CAPACITY, "n=%d outside [1,%d]", n, QJ_MAX_QUBITS);
    if (nshards < 1 || (nshards & (nshards - 1))) return fail(QJ_ERR_INVALID_ARG, "nshards=%d is not a power of two", nshards);
    if (nranks < 1 || (nranks & (nranks - 1))) return fail(QJ_ERR_INVALID_ARG, "%d ranks is not a power of two", nranks);
    const int ptot = comm ? nranks : nshards;
    int g = 0;
    while ((1 << g) < ptot) ++g;
    if (g >= n) return fail(QJ_ERR_CAPACITY, "%d shards need more than n=%d qubits", ptot, n);
    if (!shards) return fail(QJ_ERR_INVALID_ARG, "amplitude buffer is NULL");
    for (int r = 0; r < nshards; ++r) {
        if (!shards[r]) return fail(QJ_ERR_INVALID_ARG, "shard %d buffer is NULL", r);
        if (reinterpret_cast<uintptr_t>(shards[r]) & 15u)
            return fail(QJ_ERR_INVALID_ARG, "shard %d buffer is not 16-byte aligned", r);
    }
    if (basis_index != QJ_KEEP && n < 64 && basis_index >= (1ull << n))
        return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "basis_index %llu >= 2^%d", (unsigned long long)basis_index, n);
    qj_state s = new (std::nothrow) qj_state_s;
    if (!s) return fail(QJ_ERR_CAPACITY, "out of host memory");
    s->n = n;
    s->g = g;
    s->nl = n - g;
    s->dt = dt;
    s->amp_bytes = dt == QJ_C64 ? 8 : 16;
    s->shards.assign(shards, shards + nshards);
    s->stream = static_cast<cudaStream_t>(cuda_stream);
    s->comm = comm;
    s->rank = rank;
    s->nranks = nranks;
    s->host = host;
    s->phys.resize(n);
    for (int q = 0; q < n; ++q) s->phys[q] = n - 1 - q;  // reading R1
    *out = s;
    if (basis_index != QJ_KEEP) {
        qj_status st = qj_state_reset(s, basis_index);
        if (st != QJ_OK) {
            delete s;
            *out = nullptr;
            return st;
        }
    }
    return QJ_OK;
}

qj_status qj_state_init(qj_state* out, void* amps_dev, int n, qj_dtype dt, uint64_t basis_index, void* cuda_stream,
                        void* nccl_comm) {
    void* shards[1] = {amps_dev};
    if (nccl_comm == nullptr) return init_common(out, shards, 1, n, dt, basis_index, cuda_stream);
    const char* why = nullptr;
    const NcclApi* api = nccl_api(&why);
    if (!api) return fail(QJ_ERR_NCCL, "NCCL unavailable: %s", why ? why : "?");
    int rank = 0, count = 1;
    ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
    if (api->CommUserRank(comm, &rank) != ncclSuccess || api->CommCount(comm, &count) != ncclSuccess)
        return fail(QJ_ERR_NCCL, "could not query the NCCL communicator");
    return init_common(out, shards, 1, n, dt, basis_index, cuda_stream, nccl_comm, rank, count);
}

qj_status qj_state_init_sharded(qj_state* out, void* const* shards, int nshards, int n, qj_dtype dt,
                                uint64_t basis_index, void* cuda_stream) {
    return init_common(out, shards, nshards, n, dt, basis_index, cuda_stream);
}

qj_status qj_state_init_host(qj_state* out, void* amps_host, int n, qj_dtype dt, int nslices, uint64_t basis_index,
                             void* cuda_stream) {
    if (!out) return fail(QJ_ERR_INVALID_ARG, "out is NULL");
    if (!dtype_ok(dt)) return fail(QJ_ERR_DTYPE, "unknown dtype %d", (int)dt);
    if (n < 1 || n > QJ_MAX_QUBITS) return fail(QJ_ERR_CAPACITY, "n=%d outside [1,%d]", n, QJ_MAX_QUBITS);
    if (nslices < 1 || (nslices & (nslices - 1))) return fail(QJ_ERR_INVALID_ARG, "nslices=%d is not a power of two", nslices);
    if (!amps_host) return fail(QJ_ERR_INVALID_ARG, "amplitude buffer is NULL");
    int g = 0;
    while ((1 << g) < nslices) ++g;
    if (g >= n) return fail(QJ_ERR_CAPACITY, "%d slices need more than n=%d qubits", nslices, n);
    const size_t amp = dt == QJ_C64 ? 8 : 16;
    const size_t slice = amp << (n - g);
    std::vector<void*> sl((size_t)nslices);
    for (int r = 0; r < nslices; ++r) sl[(size_t)r] = static_cast<unsigned char*>(amps_host) + (size_t)r * slice;
    qj_status st = init_common(out, sl.data(), nslices, n, dt, QJ_KEEP, cuda_stream, nullptr, 0, 1, true);
    if (st != QJ_OK) return st;
    (*out)->host_base = amps_host;
    host_identity_halves(*out);
    if (basis_index != QJ_KEEP) {
        st = qj_state_reset(*out, basis_index);
        if (st != QJ_OK) {
            qj_state_free(*out);
            *out = nullptr;
        }
    }
    return st;
}

qj_status qj_state_reset(qj_state s, uint64_t basis_index) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (basis_index == QJ_KEEP) return QJ_OK;
    if (s->n < 64 && basis_index >= (1ull << s->n))
        return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "basis_index %llu >= 2^%d", (unsigned long long)basis_index, s->n);
    for (int q = 0; q < s->n; ++q) s->phys[q] = s->n - 1 - q;
    const uint64_t owner = basis_index >> s->nl;
    const uint64_t local = basis_index & ((1ull << s->nl) - 1);
    if (s->host) {  // host slices: wait for in-flight write-backs, then fill on the host
        cudaError_t e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "host reset sync");
        host_identity_halves(s);
        const size_t bytes = (size_t)s->amp_bytes << s->nl;
        for (size_t i = 0; i < s->shards.size(); ++i) std::memset(s->shards[i], 0, bytes);
        unsigned char* p = static_cast<unsigned char*>(s->shards[(size_t)owner]) + local * (size_t)s->amp_bytes;
        if (s->dt == QJ_C64) {
            const float one[2] = {1.0f, 0.0f};
            std::memcpy(p, one, sizeof(one));
        } else {
            const double one[2] = {1.0, 0.0};
            std::memcpy(p, one, sizeof(one));
        }
        return QJ_OK;
    }
    for (size_t i = 0; i < s->shards.size(); ++i) {
        const uint64_t r = s->comm ? (uint64_t)s->rank : (uint64_t)i;
        cudaError_t e = by_dtype(s->dt, [&](auto z) {
            using R = decltype(z);
            return run_init<R>(s->shards[i], s->nl, local, r == owner, s->stream, s->ls);
        });
        if (e != cudaSuccess) return cuda_fail(e, "init launch");
    }
    s->ctr.launches = s->ls.launches;
    return QJ_OK;
}

qj_status qj_set_profiling(qj_state s, int on) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    s->profiling = on != 0;
    return QJ_OK;
}

qj_status qj_get_profile(qj_state s, qj_profile_entry* out, int max_entries, int* count, int reset) {
    if (!s || !count || (max_entries > 0 && !out)) return fail(QJ_ERR_INVALID_ARG, "NULL argument");
    cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "qj_get_profile");
    uint64_t launches[PROF_N] = {};
    double ms[PROF_N] = {}, bytes[PROF_N] = {};
    for (auto& r : s->recs) {
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        launches[r.kind]++;
        ms[r.kind] += t;
        bytes[r.kind] += r.bytes;
    }
    int c = 0;
    if (reset & 2) {  // one entry per recorded launch, in enqueue order
        for (auto& r : s->recs) {
            if (c >= max_entries) break;
            float t = 0.f;
            cudaEventElapsedTime(&t, r.a, r.b);
            std::memset(&out[c], 0, sizeof(out[c]));
            std::strncpy(out[c].name, kProfNames[r.kind], sizeof(out[c].name) - 1);
            out[c].launches = 1;
            out[c].total_ms = t;
            out[c].alg_bytes = r.bytes;
            ++c;
        }
    }
    for (int k = 0; k < PROF_N && c < max_entries && !(reset & 2); ++k) {
        if (!launches[k]) continue;
        std::memset(&out[c], 0, sizeof(out[c]));
        std::strncpy(out[c].name, kProfNames[k], sizeof(out[c].name) - 1);
        out[c].launches = launches[k];
        out[c].total_ms = ms[k];
        out[c].alg_bytes = bytes[k];
        ++c;
    }
    *count = c;
    if (reset & 1) {
        for (auto& r : s->recs) {
            s->pool.push_back(r.a);
            s->pool.push_back(r.b);
        }
        s->recs.clear();
    }
    return QJ_OK;
}

qj_status qj_state_free(qj_state s) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    cudaStreamSynchronize(s->stream);
    for (auto& r : s->recs) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    for (auto ev : s->pool) cudaEventDestroy(ev);
    s->stg.release();
    for (auto* p : s->plans) release_plan(p);
    s->plans.clear();
    if (s->scratch) cudaFree(s->scratch);
    if (s->bins) cudaFree(s->bins);
    if (s->xbuf) cudaFree(s->xbuf);
    if (s->xstream) {
        cudaStreamSynchronize(s->xstream);
        for (int k = 0; k < 2; ++k) {
            cudaEventDestroy(s->xev_in[k]);
            cudaEventDestroy(s->xev_out[k]);
        }
        cudaEventDestroy(s->xev_start);
        cudaStreamDestroy(s->xstream);
    }
    if (s->mbuf) cudaFree(s->mbuf);
    if (s->hp.ready) {
        cudaStreamSynchronize(s->hp.h2d);
        cudaStreamSynchronize(s->hp.d2h);
        for (int b = 0; b < 3; ++b) {
            cudaFree(s->hp.dbuf[b]);
            cudaEventDestroy(s->hp.up[b]);
            cudaEventDestroy(s->hp.done[b]);
            cudaEventDestroy(s->hp.freed[b]);
        }
        cudaEventDestroy(s->hp.mark);
        cudaEventDestroy(s->hp.tail);
        cudaStreamDestroy(s->hp.h2d);
        cudaStreamDestroy(s->hp.d2h);
    }
    delete s;
    return QJ_OK;
}

qj_status qj_state_info(qj_state s, int* n, int* n_local, int* dtype, int* nshards) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (n) *n = s->n;
    if (n_local) *n_local = s->nl;
    if (dtype) *dtype = (int)s->dt;
    if (nshards) *nshards = s->total_shards();
    return QJ_OK;
}

qj_status qj_state_layout(qj_state s, int* phys) {
    if (!s || !phys) return fail(QJ_ERR_INVALID_ARG, "NULL argument");
    for (int q = 0; q < s->n; ++q) phys[q] = s->phys[q];
    return QJ_OK;
}

qj_status qj_get_counters(qj_state s, qj_counters* out, int reset) {
    if (!s || !out) return fail(QJ_ERR_INVALID_ARG, "NULL argument");
    s->ctr.launches = s->ls.launches;
    *out = s->ctr;
    if (reset) {
        s->ctr = qj_counters{};
        s->ls.launches = 0;
    }
    return QJ_OK;
}

static qj_status apply_one(qj_state s, int kind, const int* targets, int nt, const int* controls, int nc,
                           const void* data) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    std::vector<LGate> gs(1);
    if (qj_status st = make_lgate(s, kind, targets, nt, controls, nc, data, gs[0])) return st;
    return apply_lgates(s, gs, false);
}

qj_status qj_apply_gate(qj_state s, int n, const int* targets, int nt, const int* controls, int nc,
                        const void* matrix) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (n != s->n) return fail(QJ_ERR_INVALID_ARG, "n=%d does not match the state's n=%d", n, s->n);
    return apply_one(s, QJ_GATE_DENSE, targets, nt, controls, nc, matrix);
}

qj_status qj_apply_x(qj_state s, int target, const int* controls, int nc) {
    return apply_one(s, QJ_GATE_X, &target, 1, controls, nc, nullptr);
}

qj_status qj_apply_z(qj_state s, int target, const int* controls, int nc) {
    return apply_one(s, QJ_GATE_Z, &target, 1, controls, nc, nullptr);
}

qj_status qj_apply_swap(qj_state s, int t0, int t1, const int* controls, int nc) {
    const int t[2] = {t0, t1};
    return apply_one(s, QJ_GATE_SWAP, t, 2, controls, nc, nullptr);
}

qj_status qj_apply_fsim(qj_state s, int t0, int t1, const void* u2x2, const void* phase11, const int* controls,
                        int nc) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (!u2x2 || !phase11) return fail(QJ_ERR_INVALID_ARG, "fSim parameters are NULL");
    // pack (u00,u01,u10,u11,phase11) contiguously in the state's dtype
    const size_t cb = (size_t)s->amp_bytes;
    unsigned char buf[5 * 16];
    std::memcpy(buf, u2x2, 4 * cb);
    std::memcpy(buf + 4 * cb, phase11, cb);
    const int t[2] = {t0, t1};
    return apply_one(s, QJ_GATE_FSIM, t, 2, controls, nc, buf);
}

qj_status qj_apply_diagonal(qj_state s, const int* targets, int nt, const void* diag, const int* controls, int nc) {
    return apply_one(s, QJ_GATE_DIAG, targets, nt, controls, nc, diag);
}

qj_status qj_apply_circuit(qj_state s, const qj_gate* gates, int ngates, uint32_t flags) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (ngates < 0) return fail(QJ_ERR_INVALID_ARG, "ngates=%d < 0", ngates);
    if (ngates > 0 && !gates) return fail(QJ_ERR_INVALID_ARG, "gates is NULL");
    if (flags & ~(QJ_FUSE | QJ_FUSE_GATES | 0xF0u)) return fail(QJ_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
    if (fuse_width(flags) > 5) return fail(QJ_ERR_INVALID_ARG, "fusion width %d > 5", fuse_width(flags));
    std::vector<LGate> gs((size_t)ngates);
    for (int i = 0; i < ngates; ++i) {
        const qj_gate& g = gates[i];
        if (g.nt > QJ_MAX_TARGETS || g.nc > QJ_MAX_CONTROLS)
            return fail(QJ_ERR_TOO_MANY_TARGETS, "gate %d: nt=%d nc=%d exceeds the limits", i, g.nt, g.nc);
        qj_status st = make_lgate(s, g.kind, g.targets, g.nt, g.controls, g.nc, g.data, gs[(size_t)i]);
        if (st != QJ_OK) {
            g_err = "gate " + std::to_string(i) + ": " + g_err;
            return st;
        }
    }
    if (flags & QJ_FUSE_GATES) gs = fuse_gates(gs, s->n, fuse_width(flags));
    bool done = false;
    if (qj_status st = apply_circuit_cached(s, gates, ngates, flags, gs, &done)) return st;
    if (done) return QJ_OK;
    s->planner.auto_fuse_ = !(flags & QJ_FUSE_GATES);
    return apply_lgates(s, gs, (flags & QJ_FUSE) != 0);
}

// fp64 marginal over the listed logical qubits into s->bins[2^nq] (all-reduced
// across NCCL ranks).  Validates the qubit list.
static qj_status marginal_bins(qj_state s, const int* qubits, int nq) {
    cudaError_t e = cudaSuccess;
    const int n = s->n, nl = s->nl;
    if (nq < 1 || nq > n) return fail(QJ_ERR_INVALID_ARG, "nq=%d outside [1,%d]", nq, n);
    if (nq > 30) return fail(QJ_ERR_CAPACITY, "marginal over %d qubits is too large (max 30)", nq);
    uint64_t seen_lo = 0;
    for (int i = 0; i < nq; ++i) {
        const int q = qubits[i];
        if (q < 0 || q >= n) return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "qubit %d out of range [0,%d)", q, n);
        if (seen_lo & (1ull << q)) return fail(QJ_ERR_OVERLAPPING_QUBITS, "qubit %d listed twice", q);
        seen_lo |= 1ull << q;
    }
    const size_t nb = (size_t)1 << nq;
    if (qj_status st = ensure_bins(s, nb)) return st;
    e = cudaMemsetAsync(s->bins, 0, nb * sizeof(double), s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "bins memset");
    auto one = [&](size_t i, const void* src) -> cudaError_t {
        const uint64_t r = s->comm ? (uint64_t)s->rank : (uint64_t)i;
        int pos[64], gv[64];
        for (int k = 0; k < nq; ++k) {
            const int b = s->phys[qubits[k]];
            if (b < nl) {
                pos[k] = b;
                gv[k] = 0;
            } else {
                pos[k] = -1;
                gv[k] = (int)((r >> (b - nl)) & 1u);
            }
        }
        return by_dtype(s->dt, [&](auto z) {
            using R = decltype(z);
            return run_prob_marginal<R>(src, nl, pos, gv, nq, s->bins, s->stream, s->ls);
        });
    };
    if (s->host) {
        std::vector<int> all(s->shards.size());
        for (size_t i = 0; i < all.size(); ++i) all[i] = (int)i;
        if (qj_status q = host_sweep(s, all, false, [&](int r, void* d) { return one((size_t)r, d); })) return q;
    } else {
        for (size_t i = 0; i < s->shards.size(); ++i) {
            e = one(i, s->shards[i]);
            if (e != cudaSuccess) return cuda_fail(e, "marginal launch");
        }
    }
    if (s->comm) {  // sum the per-rank fp64 bins across ranks
        const char* why = nullptr;
        const NcclApi* api = nccl_api(&why);
        if (!api) return fail(QJ_ERR_NCCL, "NCCL unavailable: %s", why ? why : "?");
        const ncclResult_t r = api->AllReduce(s->bins, s->bins, nb, ncclFloat64, ncclSum,
                                              static_cast<ncclComm_t>(s->comm), s->stream);
        if (r != ncclSuccess) return fail(QJ_ERR_NCCL, "marginal all-reduce: %s", api->GetErrorString(r));
    }
    return QJ_OK;
}

qj_status qj_probabilities(qj_state s, const int* qubits, int nq, void* out_dev) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (!out_dev) return fail(QJ_ERR_INVALID_ARG, "out_dev is NULL");
    cudaError_t e = cudaSuccess;
    const int n = s->n, nl = s->nl;
    if (qubits == nullptr && nq == -1) {
        bool identity = true;
        for (int q = 0; q < n; ++q) identity &= (s->phys[q] == n - 1 - q);
        const size_t rb = s->dt == QJ_C64 ? 4 : 8;
        if (s->comm && !identity) {
            // rank r's output is the canonical slice [r 2^nl, (r+1) 2^nl), which a
            // remapped layout spreads over every rank: move the data back to the
            // canonical layout first (exact moves; the logical state is unchanged)
            if (qj_status st = qj_state_canonicalize(s)) return st;
            identity = true;
        }
        auto one = [&](size_t i, const void* src) -> cudaError_t {
            const uint64_t r = s->comm ? (uint64_t)s->rank : (uint64_t)i;
            if (identity) {
                // NCCL-sharded: out_dev holds this rank's 2^n_local values
                void* dst = static_cast<unsigned char*>(out_dev) + (s->comm ? 0 : rb * (r << nl));
                return by_dtype(s->dt, [&](auto z) {
                    using R = decltype(z);
                    return run_prob_full<R>(src, nl, dst, s->stream, s->ls);
                });
            }
            int cpos[64];
            for (int q = 0; q < n; ++q) cpos[s->phys[q]] = n - 1 - q;
            return by_dtype(s->dt, [&](auto z) {
                using R = decltype(z);
                return run_prob_scatter<R>(src, nl, r, n, cpos, out_dev, s->stream, s->ls);
            });
        };
        if (s->host) {
            std::vector<int> all(s->shards.size());
            for (size_t i = 0; i < all.size(); ++i) all[i] = (int)i;
            if (qj_status q = host_sweep(s, all, false, [&](int r, void* d) { return one((size_t)r, d); })) return q;
        } else {
            for (size_t i = 0; i < s->shards.size(); ++i) {
                e = one(i, s->shards[i]);
                if (e != cudaSuccess) return cuda_fail(e, "probabilities launch");
            }
        }
        s->ctr.launches = s->ls.launches;
        return QJ_OK;
    }
    if (!qubits) return fail(QJ_ERR_INVALID_ARG, "qubits is NULL (use nq=-1 for the full vector)");
    if (qj_status st = marginal_bins(s, qubits, nq)) return st;
    const size_t nb = (size_t)1 << nq;
    e = by_dtype(s->dt, [&](auto z) {
        using R = decltype(z);
        return run_bins_to_out<R>(s->bins, nb, out_dev, s->stream, s->ls);
    });
    if (e != cudaSuccess) return cuda_fail(e, "bins launch");
    s->ctr.launches = s->ls.launches;
    return QJ_OK;
}

// ------------------------------------------------------------------ measurement
static qj_status check_qubit_list(qj_state s, const int* qubits, int nq) {
    if (!qubits) return fail(QJ_ERR_INVALID_ARG, "qubits is NULL");
    if (nq < 1 || nq > s->n) return fail(QJ_ERR_INVALID_ARG, "nq=%d outside [1,%d]", nq, s->n);
    uint64_t seen = 0;
    for (int i = 0; i < nq; ++i) {
        const int q = qubits[i];
        if (q < 0 || q >= s->n) return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "qubit %d out of range [0,%d)", q, s->n);
        if (seen & (1ull << q)) return fail(QJ_ERR_OVERLAPPING_QUBITS, "qubit %d listed twice", q);
        seen |= 1ull << q;
    }
    return QJ_OK;
}

qj_status qj_collapse(qj_state s, const int* qubits, int nq, uint64_t outcome, double* prob_out) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (qj_status st = check_qubit_list(s, qubits, nq)) return st;
    if (nq < 64 && (outcome >> nq) != 0)
        return fail(QJ_ERR_INVALID_ARG, "outcome %llu >= 2^%d", (unsigned long long)outcome, nq);
    const int nl = s->nl;
    int pos[64], val[64], m = 0;
    uint64_t gmask = 0, gwant = 0, mask = 0, want = 0;
    for (int i = 0; i < nq; ++i) {
        const int b = s->phys[qubits[i]];
        const int v = (int)((outcome >> (nq - 1 - i)) & 1u);
        if (b < nl) {
            pos[m] = b;
            val[m++] = v;
            mask |= 1ull << b;
            if (v) want |= 1ull << b;
        } else {
            gmask |= 1ull << (b - nl);
            if (v) gwant |= 1ull << (b - nl);
        }
    }
    const size_t nsh = s->shards.size();
    const size_t kPartials = 2048;
    if (qj_status st = ensure_mbuf(s, (kPartials + nsh) * sizeof(double))) return st;
    double* partial = static_cast<double*>(s->mbuf);
    double* outs = partial + kPartials;
    cudaError_t e = cudaSuccess;
    std::vector<char> match(nsh);
    std::vector<int> matching;
    auto norm_one = [&](size_t i, const void* src) -> cudaError_t {
        return by_dtype(s->dt, [&](auto z) {
            using R = decltype(z);
            return run_subspace_norm<R>(src, nl, pos, val, m, partial, outs + i, s->stream, s->ls);
        });
    };
    for (size_t i = 0; i < nsh; ++i) {
        const uint64_t r = s->comm ? (uint64_t)s->rank : (uint64_t)i;
        match[i] = (r & gmask) == gwant;
        if (match[i]) {
            matching.push_back((int)i);
            e = s->host ? cudaSuccess : norm_one(i, s->shards[i]);
        } else {
            e = cudaMemsetAsync(outs + i, 0, sizeof(double), s->stream);
        }
        if (e != cudaSuccess) return cuda_fail(e, "collapse norm");
    }
    if (s->host)
        if (qj_status q = host_sweep(s, matching, false, [&](int r, void* d) { return norm_one((size_t)r, d); }))
            return q;
    if (s->comm) {
        const char* why = nullptr;
        const NcclApi* api = nccl_api(&why);
        if (!api) return fail(QJ_ERR_NCCL, "NCCL unavailable: %s", why ? why : "?");
        const ncclResult_t r = api->AllReduce(outs, outs, 1, ncclFloat64, ncclSum, static_cast<ncclComm_t>(s->comm),
                                              s->stream);
        if (r != ncclSuccess) return fail(QJ_ERR_NCCL, "collapse all-reduce: %s", api->GetErrorString(r));
    }
    std::vector<double> h(nsh);
    e = cudaMemcpyAsync(h.data(), outs, nsh * sizeof(double), cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "collapse norm readback");
    double P = 0.0;
    for (size_t i = 0; i < nsh; ++i) P += h[i];  // shard order: deterministic
    if (prob_out) *prob_out = P;
    if (!(P > 1e-14)) return fail(QJ_ERR_ZERO_PROBABILITY, "P(outcome=%llu) = %.3e <= 1e-14", (unsigned long long)outcome, P);
    const double scale = 1.0 / std::sqrt(P);
    const size_t bytes = ((size_t)s->amp_bytes) << nl;
    auto apply_one = [&](const void* dst) -> cudaError_t {
        return by_dtype(s->dt, [&](auto z) {
            using R = decltype(z);
            return run_collapse_apply<R>(const_cast<void*>(dst), nl, mask, want, scale, s->stream, s->ls);
        });
    };
    if (s->host) {  // non-matching slices are zeroed on the host (the stream is idle here)
        for (size_t i = 0; i < nsh; ++i)
            if (!match[i]) {
                std::memset(s->halves[2 * i], 0, bytes / 2);
                std::memset(s->halves[2 * i + 1], 0, bytes / 2);
            }
        if (qj_status q = host_sweep(s, matching, true, [&](int, void* d) { return apply_one(d); })) return q;
    } else {
        for (size_t i = 0; i < nsh; ++i) {
            e = match[i] ? apply_one(s->shards[i]) : cudaMemsetAsync(s->shards[i], 0, bytes, s->stream);
            if (e != cudaSuccess) return cuda_fail(e, "collapse apply");
        }
    }
    s->ctr.launches = s->ls.launches;
    return QJ_OK;
}

static qj_status sample_impl(const double* p, int nbits, uint64_t nshots, uint64_t seed, const qj_sample_opts* opts,
                             int64_t* samples, uint64_t* counts, cudaStream_t st, void* scratch, LaunchStats& ls) {
    if (!p) return fail(QJ_ERR_INVALID_ARG, "probabilities are NULL");
    if (nbits < 0 || nbits > 34) return fail(QJ_ERR_CAPACITY, "nbits=%d outside [0,34]", nbits);
    if (nshots == 0) return fail(QJ_ERR_INVALID_ARG, "nshots must be >= 1");
    if (!samples && !counts) return fail(QJ_ERR_INVALID_ARG, "samples and counts are both NULL");
    const int method = opts ? opts->method : QJ_SAMPLE_DIRECT;
    const uint64_t nb = 1ull << nbits;
    cudaError_t e = cudaSuccess;
    if (method == QJ_SAMPLE_DIRECT) {
        void* buf = scratch;
        if (!buf) {
            e = cudaMallocAsync(&buf, direct_scratch_bytes(nb), st);
            if (e != cudaSuccess) return cuda_fail(e, "sampler scratch alloc");
        }
        e = run_direct_cdf(p, nb, buf, st, ls);
        uint64_t total = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(&total, direct_total_ptr(buf, nb), sizeof(total), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e == cudaSuccess && total != 0 && total != kTotalOverflow)
            e = run_direct_shots(buf, nb, nshots, seed, samples, counts, st, ls);
        if (!scratch) cudaFreeAsync(buf, st);
        if (e != cudaSuccess) return cuda_fail(e, "direct sampler");
        if (total == kTotalOverflow)
            return fail(QJ_ERR_INVALID_ARG, "direct sampler: weights sum to >= 15.5 (normalise them; the 2^-60 fixed-point CDF holds totals below 16)");
        if (total == 0) return fail(QJ_ERR_ZERO_PROBABILITY, "all %llu probabilities are zero", (unsigned long long)nb);
        return QJ_OK;
    }
    if (method != QJ_SAMPLE_METROPOLIS && method != QJ_SAMPLE_METROPOLIS_FLIP)
        return fail(QJ_ERR_INVALID_ARG, "unknown sampling method %d", method);
    uint64_t C = opts->nchains ? opts->nchains : std::min<uint64_t>(nshots, 4096);
    const uint64_t per = (nshots + C - 1) / C;
    const uint64_t B = opts->burnin == QJ_AUTO ? std::max<uint64_t>(100, (per + 9) / 10) : opts->burnin;
    if (B >= 0xFFFFFFFFull || per >= 0xFFFFFFFFull - B)
        return fail(QJ_ERR_CAPACITY, "burn-in %llu + %llu shots per chain exceed the 2^32 - 1 step counter",
                    (unsigned long long)B, (unsigned long long)per);
    e = run_metropolis(p, nbits, nshots, seed, (uint32_t)C, B, method == QJ_SAMPLE_METROPOLIS_FLIP, samples, counts,
                       st, ls);
    if (e != cudaSuccess) return cuda_fail(e, "Metropolis sampler");
    return QJ_OK;
}

qj_status qj_sample_distribution(const double* probs_dev, int nbits, uint64_t nshots, uint64_t seed,
                                 const qj_sample_opts* opts, int64_t* samples_dev, uint64_t* counts_dev,
                                 void* stream) {
    LaunchStats ls;
    return sample_impl(probs_dev, nbits, nshots, seed, opts, samples_dev, counts_dev,
                       static_cast<cudaStream_t>(stream), nullptr, ls);
}

qj_status qj_sample(qj_state s, const int* qubits, int nq, uint64_t nshots, uint64_t seed,
                    const qj_sample_opts* opts, int64_t* samples_dev, uint64_t* counts_dev) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (qj_status st = check_qubit_list(s, qubits, nq)) return st;
    if (nshots == 0) return fail(QJ_ERR_INVALID_ARG, "nshots must be >= 1");
    if (!samples_dev && !counts_dev) return fail(QJ_ERR_INVALID_ARG, "samples and counts are both NULL");
    if (qj_status st = marginal_bins(s, qubits, nq)) return st;
    const bool direct = !opts || opts->method == QJ_SAMPLE_DIRECT;
    void* scratch = nullptr;
    if (direct) {
        if (qj_status st = ensure_mbuf(s, direct_scratch_bytes(1ull << nq))) return st;
        scratch = s->mbuf;
    }
    qj_status st = sample_impl(s->bins, nq, nshots, seed, opts, samples_dev, counts_dev, s->stream, scratch, s->ls);
    s->ctr.launches = s->ls.launches;
    return st;
}

qj_status qj_measure(qj_state s, const int* qubits, int nq, uint64_t seed, uint64_t* outcome_out, double* prob_out) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (!outcome_out) return fail(QJ_ERR_INVALID_ARG, "outcome_out is NULL");
    if (qj_status st = check_qubit_list(s, qubits, nq)) return st;
    if (qj_status st = marginal_bins(s, qubits, nq)) return st;
    const size_t sb = direct_scratch_bytes(1ull << nq);
    if (qj_status st = ensure_mbuf(s, sb + 64)) return st;
    int64_t* shot = reinterpret_cast<int64_t*>(static_cast<char*>(s->mbuf) + ((sb + 15) & ~size_t(15)));
    if (qj_status st = sample_impl(s->bins, nq, 1, seed, nullptr, shot, nullptr, s->stream, s->mbuf, s->ls)) return st;
    int64_t h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, shot, sizeof(h), cudaMemcpyDeviceToHost, s->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "measurement readback");
    *outcome_out = (uint64_t)h;
    return qj_collapse(s, qubits, nq, (uint64_t)h, prob_out);
}

// ------------------------------------------------------------------ qj_simulate
// QJ_LIVE_TILES=0 runs every later tile pass over the whole state (A/B check)
// Live-tile passes: amplitudes whose newly windowed bits not yet touched by a
// segment's register ops differ from the basis are still zero, so the JIT
// skips their transposes and arithmetic (tile_jit.cpp, zero tracking).  Put
// those still-constrained thread bits of every later segment on warp bits
// (thread-id bits >= 5; lanes 0..4 keep their bank-conflict / store roles) so
// the skips are warp-uniform.
static void live_thread_order(TileSpec& t, int amp_bytes) {
    const int M = amp_bytes == 16 ? 3 : 4;  // lanes 0..M-1: swizzle residues / the output's low bits
    uint32_t zl = 0;  // window-local zero mask
    for (int j = 0; j < TILE_W; ++j)
        if ((t.zero_mask >> t.wpos[j]) & 1) zl |= 1u << j;
    uint32_t cons = zl;
    for (size_t s = 0; s < t.segs.size(); ++s) {
        TSeg& S = t.segs[s];
        uint32_t rsel = 0;
        for (int j = 0; j < TILE_R; ++j) rsel |= 1u << S.rbits[j];
        if (s > 0) {
            // constrained thread bits to the top thread-id positions, order otherwise kept
            std::vector<int8_t> lanes(S.tbits, S.tbits + std::min(5, TILE_T)), rest, hot;
            for (int i = std::min(5, TILE_T); i < TILE_T; ++i)
                ((cons >> S.tbits[i]) & 1 ? hot : rest).push_back(S.tbits[i]);
            // a constrained lane bit moves up too when a warp position is free for it
            for (int i = std::min(5, TILE_T) - 1; i >= M && !rest.empty(); --i)
                if ((cons >> lanes[i]) & 1) {
                    hot.push_back(lanes[i]);
                    lanes[i] = rest.front();
                    rest.erase(rest.begin());
                }
            int k = 0;
            for (int8_t b : lanes) S.tbits[k++] = b;
            for (int8_t b : rest) S.tbits[k++] = b;
            for (int8_t b : hot) S.tbits[k++] = b;
        }
        cons &= ~rsel;
    }
}

static bool live_tiles_on() {
    static const bool on = !(getenv("QJ_LIVE_TILES") && getenv("QJ_LIVE_TILES")[0] == '0');
    return on;
}

// qj_simulate from |basis>: the first tile pass synthesises the one tile
// holding the basis amplitude; the run of tile passes after it runs only the
// live tiles (§5.2 "Live tiles").  Returns whether no init kernel is needed.
static bool setup_live_tiles(std::vector<Step>& steps, int nl, int amp_bytes, uint64_t basis) {
    bool init_none = false;
    Step& f = steps.front();
    f.tile.synth = true;
    f.tile.synth_index = basis;
    f.alg_bytes = 2.0 * amp_bytes * std::ldexp(1.0, TILE_W);  // one live tile (the rest: init kernel)
    // the run of tile passes after it: amplitudes whose bits outside
    // every window so far differ from |basis> are still zero, and each
    // pass maps every tile onto itself, so only the tiles whose
    // not-yet-windowed bits equal the basis bits are live
    const uint64_t all = nl >= 64 ? ~0ull : (1ull << nl) - 1;
    uint64_t windowed = 0;
    for (size_t i = 0; i < steps.size() && steps[i].type == Step::TILE && live_tiles_on(); ++i) {
        Step& t = steps[i];
        uint64_t wm = 0;
        for (int j = 0; j < TILE_W; ++j) wm |= 1ull << t.tile.wpos[j];
        if (i == 0) {  // the synthesised pass: the one tile holding x is the grid
            t.tile.fix_mask = all & ~wm;
            t.tile.fix_val = basis & t.tile.fix_mask;
        } else {
            t.tile.fix_mask = all & ~windowed & ~wm;
            t.tile.fix_val = basis & t.tile.fix_mask;
            t.tile.zero_mask = wm & ~windowed;
            t.tile.zero_val = basis & t.tile.zero_mask;
            if (!(getenv("QJ_ZSPARSE") && getenv("QJ_ZSPARSE")[0] == '0')) live_thread_order(t.tile, amp_bytes);
            const int fb = __builtin_popcountll(t.tile.fix_mask), z = __builtin_popcountll(t.tile.zero_mask);
            t.alg_bytes = amp_bytes * (std::ldexp(1.0, nl - fb - z) + std::ldexp(1.0, nl - fb));
            // each pass reads only amplitudes the previous one wrote: once a
            // pass writes every tile, no amplitude is read before it is written
            if (!t.tile.fix_mask) init_none = true;
        }
        windowed |= wm;
    }
    return init_none;
}
static qj_status run_sim(qj_state s, qj_state_s::CachedPlan& p) {
    cudaError_t e = cudaSuccess;
    const size_t nb = p.nq > 0 ? (size_t)1 << p.nq : 0;
    if (nb) e = cudaMemsetAsync(p.sim_bins, 0, nb * sizeof(double), s->stream);
    {
        // |basis> before the circuit: written by the init kernel, or -- when the
        // first step is a tile pass that synthesises the one tile holding the
        // basis amplitude -- zeros here and that tile there (every other tile
        // of |basis> is zero in and zero out); nothing at all when a later
        // live-tile pass writes every tile before any amplitude outside the
        // tiles written so far is read (init_none)
        if (!p.init_none) {
            ProfScope prof(s, PROF_INIT, (double)s->amp_bytes * std::ldexp(1.0, s->nl));
            if (e == cudaSuccess)
                e = by_dtype(s->dt, [&](auto z) {
                    using R = decltype(z);
                    return run_init<R>(s->shards[0], s->nl, p.basis, p.init_first, s->stream, s->ls);
                });
        }
    }
    if (e != cudaSuccess) return cuda_fail(e, "simulate prologue");
    if (qj_status q = run_cached(s, p)) return q;
    if (nb && !p.marg_last) {
        int gv[16] = {};
        e = by_dtype(s->dt, [&](auto z) {
            using R = decltype(z);
            return run_prob_marginal<R>(s->shards[0], s->nl, p.qpos, gv, p.nq, p.sim_bins, s->stream, s->ls);
        });
        if (e != cudaSuccess) return cuda_fail(e, "simulate marginal");
    }
    return QJ_OK;
}
// the bins -> caller's output conversion stays outside the cached graph, so
// the output pointer is not part of the plan key (callers may pass a fresh
// buffer every call)
static qj_status run_sim_out(qj_state s, qj_state_s::CachedPlan& p, void* out) {
    const size_t nb = p.nq > 0 ? (size_t)1 << p.nq : 0;
    if (!nb) return QJ_OK;
    cudaError_t e = by_dtype(s->dt, [&](auto z) {
        using R = decltype(z);
        return run_bins_to_out<R>(p.sim_bins, nb, out, s->stream, s->ls);
    });
    if (e != cudaSuccess) return cuda_fail(e, "simulate readout");
    return QJ_OK;
}

qj_status qj_simulate(qj_state s, uint64_t basis, const qj_gate* gates, int ngates, uint32_t flags, const int* qubits,
                      int nq, void* out_dev) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    if (s->n < 64 && basis >= (1ull << s->n))
        return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "basis_index %llu >= 2^%d", (unsigned long long)basis, s->n);
    if (ngates < 0 || (ngates > 0 && !gates)) return fail(QJ_ERR_INVALID_ARG, "bad gate list");
    if (flags & ~(QJ_FUSE | QJ_FUSE_GATES | 0xF0u)) return fail(QJ_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
    if (fuse_width(flags) > 5) return fail(QJ_ERR_INVALID_ARG, "fusion width %d > 5", fuse_width(flags));
    if (nq < 0) return fail(QJ_ERR_INVALID_ARG, "nq=%d < 0", nq);
    if (nq > 0) {
        if (!out_dev) return fail(QJ_ERR_INVALID_ARG, "out_dev is NULL");
        if (qj_status st = check_qubit_list(s, qubits, nq)) return st;
    }
    const bool fast = !s->comm && !s->host && s->shards.size() == 1 && (flags & QJ_FUSE) && nq <= 10 &&
                      s->cache_on && tile_jit_available();
    if (!fast) {  // the three calls it stands for
        if (qj_status st = qj_state_reset(s, basis)) return st;
        if (qj_status st = qj_apply_circuit(s, gates, ngates, flags)) return st;
        return nq > 0 ? qj_probabilities(s, qubits, nq, out_dev) : QJ_OK;
    }
    std::vector<LGate> gs((size_t)ngates);
    for (int i = 0; i < ngates; ++i) {
        const qj_gate& g = gates[i];
        if (g.nt > QJ_MAX_TARGETS || g.nc > QJ_MAX_CONTROLS)
            return fail(QJ_ERR_TOO_MANY_TARGETS, "gate %d: nt=%d nc=%d exceeds the limits", i, g.nt, g.nc);
        if (qj_status st = make_lgate(s, g.kind, g.targets, g.nt, g.controls, g.nc, g.data, gs[(size_t)i])) {
            g_err = "gate " + std::to_string(i) + ": " + g_err;
            return st;
        }
    }
    for (int q = 0; q < s->n; ++q) s->phys[q] = s->n - 1 - q;  // the reset's map
    std::vector<uint64_t> key = plan_key(s, gates, ngates, flags);
    key.push_back(0x5117ull);
    key.push_back(basis);
    key.push_back((uint64_t)nq);
    for (int i = 0; i < nq; ++i) key.push_back((uint64_t)qubits[i]);
    qj_state_s::CachedPlan* p = nullptr;
    for (size_t i = 0; i < s->plans.size() && !p; ++i)
        if (s->plans[i]->key == key) {
            p = s->plans[i];
            std::rotate(s->plans.begin(), s->plans.begin() + (long)i, s->plans.begin() + (long)i + 1);
        }
    if (!p) {
        if (flags & QJ_FUSE_GATES) gs = fuse_gates(gs, s->n, fuse_width(flags));
        p = new qj_state_s::CachedPlan;
        p->key.swap(key);
        p->sim = true;
        p->basis = basis;
        p->nq = nq;
        PlanContext ctx{s->n, s->nl, s->g, s->amp_bytes, 1, &s->phys};
        s->planner.auto_fuse_ = !(flags & QJ_FUSE_GATES);
        s->planner.plan(ctx, gs, true, p->steps);
        p->phys_after = s->phys;
        for (int i = 0; i < nq; ++i) p->qpos[i] = p->phys_after[qubits[i]];
        const bool first_tile = !p->steps.empty() && p->steps.front().type == Step::TILE;
        const bool last_tile = !p->steps.empty() && p->steps.back().type == Step::TILE;
        p->init_first = !first_tile;
        if (first_tile) p->init_none = setup_live_tiles(p->steps, s->nl, s->amp_bytes, basis);
        if (nq > 0) {
            cudaError_t e = cudaMalloc(&p->sim_bins, sizeof(double) << nq);
            if (e != cudaSuccess) {
                release_plan(p);
                return cuda_fail(e, "simulate bins");
            }
        }
        bool in_window = last_tile;
        if (last_tile)
            for (int i = 0; i < nq; ++i) {
                bool w = false;
                for (int j = 0; j < TILE_W; ++j) w |= p->steps.back().tile.wpos[j] == p->qpos[i];
                in_window &= w;
            }
        // bins depend on (thread, register) only when every readout bit is in the
        // last window; otherwise on the tile too (per-CTA SMEM bins, nq <= 10)
        if (nq > 0 && last_tile && (in_window || nq <= 10)) {
            Step& l = p->steps.back();
            l.tile.nbins_q = nq;
            for (int i = 0; i < nq; ++i) l.tile.bin_pos[i] = (int8_t)p->qpos[i];
            l.tile.bins = p->sim_bins;
            p->marg_last = true;
        }
        for (const Step& st : p->steps) {
            if (st.type == Step::TILE) {
                PreparedTile t;
                cudaError_t e = by_dtype(s->dt, [&](auto z) {
                    using R = decltype(z);
                    return tile_prepare<R>(st.tile, s->shards[0], s->nl, t);
                });
                if (e != cudaSuccess || ((st.tile.synth || st.tile.nbins_q || st.tile.fix_mask || st.tile.zero_mask) && !t.jit)) {
                    tile_release(t);
                    release_plan(p);
                    return e != cudaSuccess ? cuda_fail(e, "tile prepare") : fail(QJ_ERR_CUDA, "simulate: JIT unavailable");
                }
                p->tiles.push_back(std::move(t));
            } else if (st.type == Step::SMALL) {
                PreparedSmall t;
                cudaError_t e = by_dtype(s->dt, [&](auto z) {
                    using R = decltype(z);
                    return small_prepare<R>(st.prog, s->shards[0], s->nl, t);
                });
                if (e != cudaSuccess) {
                    small_release(t);
                    release_plan(p);
                    return cuda_fail(e, "small prepare");
                }
                p->smalls.push_back(t);
            } else if (st.type == Step::PASS && st.pass.k > 5 && st.pass.kind == PK_DENSE) {
                p->graphable = false;
                const size_t need = (size_t)s->amp_bytes * ((size_t)1 << (2 * st.pass.k));
                if (qj_status q = ensure_scratch(s, need)) {
                    release_plan(p);
                    return q;
                }
            }
        }
        s->plans.insert(s->plans.begin(), p);
        while (s->plans.size() > 16) {
            release_plan(s->plans.back());
            s->plans.pop_back();
        }
        const uint64_t before = s->ls.launches;
        if (qj_status q = run_sim(s, *p)) return q;
        p->kernels = s->ls.launches - before;
        if (qj_status q = run_sim_out(s, *p, out_dev)) return q;
        p->uses = 1;
    } else {
        const uint64_t before = s->ls.launches;
        const bool graph_ok = p->graphable && !s->profiling && s->stream != nullptr;
        if (graph_ok && !p->exec) {
            cudaGraph_t g = nullptr;
            cudaError_t e = cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) return cuda_fail(e, "graph capture");
            qj_status q = run_sim(s, *p);
            e = cudaStreamEndCapture(s->stream, &g);
            if (q != QJ_OK) return q;
            if (e != cudaSuccess) return cuda_fail(e, "graph capture end");
            e = cudaGraphInstantiate(&p->exec, g, 0);
            cudaGraphDestroy(g);
            if (e != cudaSuccess) {
                p->exec = nullptr;
                p->graphable = false;
                cudaGetLastError();
                return cuda_fail(e, "graph instantiate");
            }
            s->ls.launches = before;
        }
        if (graph_ok && p->exec) {
            cudaError_t e = cudaGraphLaunch(p->exec, s->stream);
            if (e != cudaSuccess) return cuda_fail(e, "graph launch");
            s->ls.launches += p->kernels;
        } else if (qj_status q = run_sim(s, *p)) {
            return q;
        }
        if (qj_status q = run_sim_out(s, *p, out_dev)) return q;
        p->uses++;
    }
    account(s, *p);
    s->phys = p->phys_after;
    s->ctr.launches = s->ls.launches;
    return QJ_OK;
}

qj_status qj_fuse_circuit(int n, const qj_gate* in, int nin, int max_qubits, qj_gate* out, double* mats, int max_out,
                          int* nout, int* src) {
    if (!nout || (nin > 0 && !in) || (max_out > 0 && (!out || !mats))) return fail(QJ_ERR_INVALID_ARG, "NULL argument");
    if (n < 1 || n > QJ_MAX_QUBITS) return fail(QJ_ERR_CAPACITY, "n=%d outside [1,%d]", n, QJ_MAX_QUBITS);
    if (max_qubits < 1 || max_qubits > 5) return fail(QJ_ERR_UNSUPPORTED, "max_qubits must be in 1..5 (got %d)", max_qubits);
    const size_t stride = (size_t)2 << (2 * max_qubits);  // 2 * 4^max_qubits doubles per output gate
    qj_state_s tmp;
    tmp.n = n;
    tmp.dt = QJ_C128;
    std::vector<LGate> gs((size_t)nin);
    for (int i = 0; i < nin; ++i) {
        const qj_gate& q = in[i];
        if (q.nt > QJ_MAX_TARGETS || q.nc > QJ_MAX_CONTROLS)
            return fail(QJ_ERR_TOO_MANY_TARGETS, "gate %d: nt=%d nc=%d exceeds the limits", i, q.nt, q.nc);
        qj_status st = make_lgate(&tmp, q.kind, q.targets, q.nt, q.controls, q.nc, q.data, gs[(size_t)i]);
        if (st != QJ_OK) return st;
    }
    std::vector<LGate> fused = fuse_gates(gs, n, max_qubits);
    if ((int)fused.size() > max_out) return fail(QJ_ERR_CAPACITY, "%zu fused gates > %d", fused.size(), max_out);
    for (size_t i = 0; i < fused.size(); ++i) {
        if (src) src[i] = fused[i].src;
        const LGate& f = fused[i];
        qj_gate& o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.kind = f.kind;
        o.nt = f.nt;
        o.nc = f.nc;
        for (int j = 0; j < f.nt; ++j) o.targets[j] = f.t[j];
        for (int j = 0; j < f.nc; ++j) o.controls[j] = f.c[j];
        if (f.src >= 0) {  // a gate copied unchanged
            o.data = in[f.src].data;
        } else {
            double* m = mats + stride * i;
            for (size_t j = 0; j < f.data.size(); ++j) {
                m[2 * j] = f.data[j].real();
                m[2 * j + 1] = f.data[j].imag();
            }
            o.data = m;
        }
    }
    *nout = (int)fused.size();
    return QJ_OK;
}

void qj_exchange_peer(int rank, int gbit, int* peer, int* half_bit) {
    const ExchangeSpec e = exchange_spec(rank, gbit);
    if (peer) *peer = e.peer;
    if (half_bit) *half_bit = e.half_bit;
}

qj_status qj_plan_circuit(int n, int nshards, int amp_bytes, const qj_gate* gates, int ngates, uint32_t flags,
                          qj_plan_step* out, int max_steps, int* nsteps, int* phys) {
    if (!nsteps || (max_steps > 0 && !out)) return fail(QJ_ERR_INVALID_ARG, "NULL output");
    if (n < 1 || n > QJ_MAX_QUBITS) return fail(QJ_ERR_CAPACITY, "n=%d outside [1,%d]", n, QJ_MAX_QUBITS);
    if (nshards < 1 || (nshards & (nshards - 1))) return fail(QJ_ERR_INVALID_ARG, "nshards=%d is not a power of two", nshards);
    if (ngates < 0 || (ngates > 0 && !gates)) return fail(QJ_ERR_INVALID_ARG, "bad gate list");
    if (flags & ~QJ_FUSE) return fail(QJ_ERR_INVALID_ARG, "unknown flags 0x%x", flags);
    qj_state_s tmp;  // host-only view: n, dtype complex128
    tmp.n = n;
    tmp.dt = QJ_C128;
    int g = 0;
    while ((1 << g) < nshards) ++g;
    if (g >= n) return fail(QJ_ERR_CAPACITY, "%d shards need more than n=%d qubits", nshards, n);
    std::vector<LGate> gs((size_t)ngates);
    for (int i = 0; i < ngates; ++i) {
        const qj_gate& q = gates[i];
        if (q.nt > QJ_MAX_TARGETS || q.nc > QJ_MAX_CONTROLS)
            return fail(QJ_ERR_TOO_MANY_TARGETS, "gate %d: nt=%d nc=%d exceeds the limits", i, q.nt, q.nc);
        qj_status st = make_lgate(&tmp, q.kind, q.targets, q.nt, q.controls, q.nc, q.data, gs[(size_t)i]);
        if (st != QJ_OK) return st;
    }
    std::vector<int> map(n);
    for (int q = 0; q < n; ++q) map[q] = n - 1 - q;
    PlanContext ctx{n, n - g, g, amp_bytes, nshards, &map};
    std::vector<Step> steps;
    Planner pl;
    pl.auto_fuse_ = true;
    pl.plan(ctx, gs, (flags & QJ_FUSE) != 0, steps);
    if ((int)steps.size() > max_steps) return fail(QJ_ERR_CAPACITY, "plan has %zu steps > %d", steps.size(), max_steps);
    for (size_t i = 0; i < steps.size(); ++i) {
        const Step& st = steps[i];
        qj_plan_step& o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.type = (int)st.type;
        o.shard = st.shard;
        o.gbit = st.gbit;
        o.lbit = st.lbit;
        o.alg_bytes = st.alg_bytes;
        if (st.type != Step::PASS) continue;
        const Pass& p = st.pass;
        o.kind = p.kind;
        o.k = p.k;
        for (int j = 0; j < p.k; ++j) o.tpos[j] = p.tpos[j];
        o.nfix = p.nfix;
        for (int j = 0; j < p.nfix; ++j) {
            o.fpos[j] = p.fpos[j];
            o.fval[j] = p.fval[j];
        }
        o.touch = p.touch;
        if (p.m.size() > 256) return fail(QJ_ERR_UNSUPPORTED, "plan export: payload of %zu values", p.m.size());
        o.nm = (int)p.m.size();
        for (size_t j = 0; j < p.m.size(); ++j) {
            o.m[2 * j] = p.m[j].real();
            o.m[2 * j + 1] = p.m[j].imag();
        }
    }
    *nsteps = (int)steps.size();
    if (phys)
        for (int q = 0; q < n; ++q) phys[q] = map[q];
    return QJ_OK;
}

// Steps that bring the logical->physical map `phys` back to canonical
// (qubit q at bit n-1-q) on `nshards` shards of 2^nl amplitudes: local pairs
// by SWAP passes on EVERY shard index (each rank runs its own), local/global
// pairs by one exchange, global pairs by three exchanges through the top
// local bit.  `phys` is updated to the canonical map.
static std::vector<Step> canonicalize_steps(int n, int nl, int nshards, int amp_bytes, std::vector<int>& phys) {
    std::vector<Step> steps;
    for (int q = 0; q < n; ++q) {
        const int want = n - 1 - q, cur = phys[q];
        if (cur == want) continue;
        int q2 = 0;
        while (phys[q2] != want) ++q2;
        if (cur < nl && want < nl) {
            for (int r = 0; r < nshards; ++r) {
                Step st;
                st.type = Step::PASS;
                st.shard = r;
                st.pass.kind = PK_SWAP;
                st.pass.k = 2;
                st.pass.tpos[0] = cur;
                st.pass.tpos[1] = want;
                st.alg_bytes = pass_alg_bytes(st.pass, nl, amp_bytes);
                steps.push_back(std::move(st));
            }
        } else if (cur >= nl && want >= nl) {
            // two global bits trade places: (a L)(b L)(a L) = (a b) through the
            // top local bit (zero-copy relabels for host-staged states)
            for (int t = 0; t < 3; ++t) {
                Step st;
                st.type = Step::EXCHANGE;
                st.gbit = (t == 1 ? want : cur) - nl;
                st.lbit = nl - 1;
                steps.push_back(std::move(st));
            }
        } else {
            Step st;
            st.type = Step::EXCHANGE;
            st.gbit = std::max(cur, want) - nl;
            st.lbit = std::min(cur, want);
            steps.push_back(std::move(st));
        }
        phys[q] = want;
        phys[q2] = cur;
    }
    return steps;
}

qj_status qj_state_canonicalize(qj_state s) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    std::vector<int> phys = s->phys;
    // total_shards(): an NCCL rank holds one shard but plans for all of them
    // (execute() runs the steps of its own shard index only)
    const std::vector<Step> steps = canonicalize_steps(s->n, s->nl, s->total_shards(), s->amp_bytes, phys);
    qj_status st = execute(s, steps);
    if (st == QJ_OK) s->phys = phys;
    if (st == QJ_OK && s->host) {  // put the half-slices back in the caller's buffer order
        cudaError_t e = cudaStreamSynchronize(s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "canonicalize sync");
        st = host_materialize(s);
    }
    return st;
}

qj_status qj_plan_canonicalize(int n, int nshards, const int* phys_in, qj_plan_step* out, int max_steps,
                               int* nsteps) {
    if (!phys_in || !nsteps || (max_steps > 0 && !out)) return fail(QJ_ERR_INVALID_ARG, "NULL argument");
    if (n < 1 || n > QJ_MAX_QUBITS) return fail(QJ_ERR_CAPACITY, "n=%d outside [1,%d]", n, QJ_MAX_QUBITS);
    if (nshards < 1 || (nshards & (nshards - 1))) return fail(QJ_ERR_INVALID_ARG, "nshards=%d is not a power of two", nshards);
    int g = 0;
    while ((1 << g) < nshards) ++g;
    if (g >= n) return fail(QJ_ERR_CAPACITY, "%d shards need more than n=%d qubits", nshards, n);
    std::vector<int> phys(phys_in, phys_in + n);
    std::vector<int> seen(n, 0);
    for (int q = 0; q < n; ++q) {
        if (phys[q] < 0 || phys[q] >= n || seen[phys[q]]++) return fail(QJ_ERR_INVALID_ARG, "phys is not a permutation of 0..n-1");
    }
    const std::vector<Step> steps = canonicalize_steps(n, n - g, nshards, 16, phys);
    if ((int)steps.size() > max_steps) return fail(QJ_ERR_CAPACITY, "plan has %zu steps > %d", steps.size(), max_steps);
    for (size_t i = 0; i < steps.size(); ++i) {
        const Step& st = steps[i];
        qj_plan_step& o = out[i];
        std::memset(&o, 0, sizeof(o));
        o.type = (int)st.type;
        o.shard = st.shard;
        o.gbit = st.gbit;
        o.lbit = st.lbit;
        o.alg_bytes = st.alg_bytes;
        if (st.type == Step::PASS) {
            o.kind = st.pass.kind;
            o.k = st.pass.k;
            for (int j = 0; j < st.pass.k; ++j) o.tpos[j] = st.pass.tpos[j];
            o.touch = st.pass.touch;
        }
    }
    *nsteps = (int)steps.size();
    return QJ_OK;
}

qj_status qj_debug_tile_sources(int n, int amp_bytes, const qj_gate* gates, int ngates, uint32_t flags,
                                const char* dir, int compile, int* nkernels) {
    if (!nkernels || (ngates > 0 && !gates)) return fail(QJ_ERR_INVALID_ARG, "NULL argument");
    if (amp_bytes != 8 && amp_bytes != 16) return fail(QJ_ERR_DTYPE, "amp_bytes must be 8 or 16");
    if (n < 1 || n > QJ_MAX_QUBITS) return fail(QJ_ERR_CAPACITY, "n=%d outside [1,%d]", n, QJ_MAX_QUBITS);
    qj_state_s tmp;
    tmp.n = n;
    tmp.dt = amp_bytes == 16 ? QJ_C128 : QJ_C64;
    std::vector<LGate> gs((size_t)ngates);
    for (int i = 0; i < ngates; ++i) {
        const qj_gate& q = gates[i];
        if (q.nt > QJ_MAX_TARGETS || q.nc > QJ_MAX_CONTROLS)
            return fail(QJ_ERR_TOO_MANY_TARGETS, "gate %d: nt=%d nc=%d exceeds the limits", i, q.nt, q.nc);
        if (qj_status st = make_lgate(&tmp, q.kind, q.targets, q.nt, q.controls, q.nc, q.data, gs[(size_t)i])) return st;
    }
    if (flags & QJ_FUSE_GATES) gs = fuse_gates(gs, n, fuse_width(flags));
    std::vector<int> map(n);
    for (int q = 0; q < n; ++q) map[q] = n - 1 - q;
    PlanContext ctx{n, n, 0, amp_bytes, 1, &map};
    std::vector<Step> steps;
    Planner pl;
    pl.auto_fuse_ = !(flags & QJ_FUSE_GATES);
    pl.plan(ctx, gs, true, steps);
    if (const char* e = getenv("QJ_DEBUG_LIVE"); e && !steps.empty() && steps.front().type == Step::TILE)
        setup_live_tiles(steps, n, amp_bytes, strtoull(e, nullptr, 0));  // the qj_simulate form from |basis>
    int k = 0;
    for (const Step& st : steps) {
        if (st.type != Step::TILE) continue;
        std::string path = dir ? std::string(dir) + "/qj_tile_" + std::to_string(k) + ".cu" : std::string();
        std::string err;
        const bool ok = amp_bytes == 16 ? tile_jit_debug_source<double>(st.tile, n, dir ? path.c_str() : nullptr, compile != 0, &err)
                                        : tile_jit_debug_source<float>(st.tile, n, dir ? path.c_str() : nullptr, compile != 0, &err);
        if (!ok) return fail(QJ_ERR_UNSUPPORTED, "tile pass %d: %s", k, err.c_str());
        ++k;
    }
    *nkernels = k;
    return QJ_OK;
}

qj_status qj_debug_nccl_self_exchange(qj_state s, int local_bit) {
    if (!s || !s->comm) return fail(QJ_ERR_INVALID_ARG, "needs an NCCL-backed state");
    if (local_bit < 0 || local_bit >= s->nl) return fail(QJ_ERR_INDEX_OUT_OF_RANGE, "local bit %d", local_bit);
    ExchangeSpec ex;
    ex.peer = s->rank;  // this rank trades the half with itself: the state must come back unchanged
    ex.half_bit = 1;
    return nccl_exchange_with(s, ex, local_bit);
}

qj_status qj_sync(qj_state s) {
    if (!s) return fail(QJ_ERR_INVALID_ARG, "state is NULL");
    cudaError_t e = cudaStreamSynchronize(s->stream);
    if (e != cudaSuccess) return cuda_fail(e, "qj_sync");
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "qj_sync");
    if (tile_check_failed()) return fail(QJ_ERR_CUDA, "qj_sync: a checked tile kernel (QJ_JIT_CHECK=1) caught an out-of-bounds access");
    return QJ_OK;
}

}  // extern "C"
