// tile_plan.cpp -- fused planning (QJ_FUSE): pack consecutive gates into
// window tile passes (tile.h), one HBM round trip per pass.
//
// Rules ("tile pass"):
//  * an uncontrolled SWAP is a relabelling of two physical bits (the handle's
//    logical->physical map; readout stays canonical through the map);
//  * a diagonal gate (<= 3 targets) becomes phase terms on any bits -- it never
//    widens the window;
//  * a 1- or 2-target non-diagonal gate must have its targets in the window;
//    the window grows (up to TILE_W bits, always including the low L bits that
//    make 128-byte contiguous runs) until a gate does not fit, which closes
//    the pass;
//  * anything else (>= 3-target non-diagonal, > 3-target diagonal) closes the
//    pass and runs as a single-gate pass.
// Inside a pass, gates are split into segments of 4 register bits; diagonal
// terms are deferred (they commute with every gate not targeting their bits)
// and flushed into a RUN just before the first gate that targets one of their
// bits, or at the end of the pass.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "planner.h"

namespace qj {

namespace {

constexpr int kMaxOpsPerPass = TILE_MAXOPS - 16;
constexpr int kMaxMatPerPass = TILE_MAXMAT;

int popc(uint64_t x) { return __builtin_popcountll(x); }

bool is_diag(const std::vector<cd>& m, int D) {
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c)
            if (r != c && m[(size_t)r * D + c] != cd(0, 0)) return false;
    return true;
}

struct Item {
    bool diag = false;
    std::vector<HTerm> terms;  // diag
    HOp op;                    // non-diag
    uint64_t tmask = 0;        // non-diag target bits
};

struct PassBuild {
    std::vector<Item> items;
    std::vector<std::vector<Step>> singles;  // each gate as single-gate passes (one per shard it touches)
    uint64_t W = 0;
    int nops = 0, nmat = 0, nterms = 0, nnd = 0;  // nnd: non-diagonal ops (each may flush one run)
    double cost = 0;                               // estimated arithmetic per amplitude
};

// Estimated arithmetic per amplitude of a tile op (FP operations; a flushed
// phase run before a non-diagonal op adds ~1 complex multiply), used to keep a
// pass's compute within its HBM time.
double op_cost(const HOp& op) {
    // dense U1 / U2: 2 FMAs per output amplitude per nonzero matrix component
    // (the JIT kernels skip zero real / imaginary parts: RX, RY, fSim)
    auto nzc = [&](int count) {
        double c = 0;
        for (int e = 0; e < count; ++e) c += (op.m[e].real() != 0) + (op.m[e].imag() != 0);
        return c;
    };
    switch (op.type) {
        case TO_X:
        case TO_SWAP: return 1 + 4;
        case TO_U2: return nzc(16) / 2 + 4;
        default: break;
    }
    const bool h = op.m.size() == 4 && op.cmask == 0 && op.m[0] == op.m[1] && op.m[0] == op.m[2] &&
                   op.m[3] == -op.m[0] && op.m[0].imag() == 0;
    return h ? 2 + 4 : nzc(4) + 4;
}

// Phase terms of a diagonal gate on physical positions.
bool diag_terms(const LGate& g, const std::vector<int>& phys, std::vector<HTerm>& out) {
    std::vector<cd> d;
    const int k = g.nt;
    if (g.kind == QJ_GATE_Z) {
        d = {cd(1, 0), cd(-1, 0)};
    } else if (g.kind == QJ_GATE_DIAG) {
        d = g.data;
    } else if (g.kind == QJ_GATE_DENSE && is_diag(g.data, 1 << k)) {
        d.resize((size_t)1 << k);
        for (int i = 0; i < (1 << k); ++i) d[i] = g.data[(size_t)i * (1 << k) + i];
    } else {
        return false;
    }
    if (k > 3) return false;
    uint64_t cm = 0;
    for (int i = 0; i < g.nc; ++i) cm |= 1ull << phys[g.c[i]];
    for (int e = 0; e < (1 << k); ++e) {
        if (d[e] == cd(1, 0)) continue;
        HTerm t;
        t.mask = cm;
        t.val = cm;
        for (int i = 0; i < k; ++i) {
            const uint64_t b = 1ull << phys[g.t[i]];
            t.mask |= b;
            if ((e >> (k - 1 - i)) & 1) t.val |= b;
        }
        t.f = d[e];
        out.push_back(t);
    }
    return true;
}

// Non-diagonal 1q/2q gate as a tile op.
bool make_op(const LGate& g, const std::vector<int>& phys, HOp& op) {
    if (g.nt > 2) return false;
    op = HOp();
    for (int i = 0; i < g.nc; ++i) op.cmask |= 1ull << phys[g.c[i]];
    for (int i = 0; i < g.nt; ++i) op.t[i] = phys[g.t[i]];
    switch (g.kind) {
        case QJ_GATE_X:
            op.type = TO_X;
            return true;
        case QJ_GATE_SWAP:
            op.type = TO_SWAP;
            return true;
        case QJ_GATE_FSIM:
            op.type = TO_U2;
            op.m.assign(16, cd(0, 0));
            op.m[0] = 1;
            op.m[5] = g.data[0];
            op.m[6] = g.data[1];
            op.m[9] = g.data[2];
            op.m[10] = g.data[3];
            op.m[15] = g.data[4];
            return true;
        case QJ_GATE_DENSE:
            op.type = g.nt == 1 ? TO_U1 : TO_U2;
            op.m = g.data;
            return true;
        default:
            return false;
    }
}

// Choose the thread-bit order of a segment: lanes 0..M-1 on window bits of
// distinct residues mod M (the swizzle period: conflict-free SMEM), or the C
// low bits first when the segment touches HBM.
void thread_bits(uint32_t rsel, int C, int M, bool global, int8_t* tb) {
    std::vector<int> avail;
    for (int j = 0; j < TILE_W; ++j)
        if (!((rsel >> j) & 1)) avail.push_back(j);
    std::vector<int> order;
    auto take = [&](int j) {
        order.push_back(j);
        avail.erase(std::find(avail.begin(), avail.end(), j));
    };
    if (global) {
        for (int j = 0; j < C; ++j) take(j);  // low window bits on lanes 0..C-1
    } else {
        for (int res = 0; res < M; ++res) {
            for (int j : avail)
                if (j % M == res) {
                    take(j);
                    break;
                }
        }
    }
    for (int j : std::vector<int>(avail)) take(j);
    for (int i = 0; i < TILE_T; ++i) tb[i] = (int8_t)order[i];
}

}  // namespace

// Build the TileSpec of one pass.
// carried (optional): diagonal items whose terms are all still pending at the
// end of the pass and touch a bit outside the window are left out of the pass
// and returned, so the caller can move them to the front of the next pass
// (they commute with everything in between).
static bool build_tile(const PassBuild& pb, int nl, int C, int M, TileSpec& ts, std::vector<int>* carried = nullptr,
                       bool final_pass = false) {
    // window: pad to TILE_W bits with unused local bits -- the lowest ones
    // (QJ_TILE_PAD=low: longer contiguous HBM rows) or the highest (default)
    uint64_t W = pb.W;
    static const bool pad_low = getenv("QJ_TILE_PAD") && getenv("QJ_TILE_PAD")[0] == 'l';
    if (pad_low) {
        for (int b = 0; b < nl && popc(W) < TILE_W; ++b) W |= 1ull << b;
    } else {
        for (int b = nl - 1; b >= 0 && popc(W) < TILE_W; --b) W |= 1ull << b;
    }
    if (popc(W) != TILE_W) return false;
    ts = TileSpec();
    ts.w = TILE_W;
    int loc[64];
    for (int b = 0, j = 0; b < 64; ++b) {
        loc[b] = -1;
        if ((W >> b) & 1) {
            ts.wpos[j] = b;
            loc[b] = j++;
        }
    }
    const uint32_t lowsel = (1u << C) - 1u;  // window-local low bits (the HBM runs)
    struct SegB {
        uint32_t rsel = 0;  // window-local register bits
        std::vector<HOp> ops;
    };
    std::vector<SegB> segs(1);
    std::vector<HTerm> pending;
    std::vector<int> pend_src;                    // item of each pending term
    std::vector<char> touched(pb.items.size(), 0);  // an item's term went into a run
    std::vector<char> skip(pb.items.size(), 0);     // carried items (final flush only)
    auto flush = [&](uint64_t conflict_mask, bool all) {
        HOp run;
        run.type = TO_RUN;
        std::vector<HTerm> keep;
        std::vector<int> keep_src;
        for (size_t i = 0; i < pending.size(); ++i) {
            const HTerm& t = pending[i];
            if (skip[pend_src[i]]) continue;
            if (all || (t.mask & conflict_mask)) {
                run.terms.push_back(t);
                touched[pend_src[i]] = 1;
            } else {
                keep.push_back(t);
                keep_src.push_back(pend_src[i]);
            }
        }
        pending.swap(keep);
        pend_src.swap(keep_src);
        if (!run.terms.empty()) segs.back().ops.push_back(std::move(run));
    };
    for (size_t ii = 0; ii < pb.items.size(); ++ii) {
        const Item& it = pb.items[ii];
        if (it.diag) {
            pending.insert(pending.end(), it.terms.begin(), it.terms.end());
            pend_src.insert(pend_src.end(), it.terms.size(), (int)ii);
            continue;
        }
        uint32_t tsel = 0;
        for (int i = 0; i < (it.op.type == TO_U1 || it.op.type == TO_X ? 1 : 2); ++i) tsel |= 1u << loc[it.op.t[i]];
        SegB& cur = segs.back();
        const bool first = segs.size() == 1;
        if ((tsel & ~cur.rsel) != 0) {
            const uint32_t want = cur.rsel | tsel;
            const bool fits = popc(want) <= TILE_R && !(first && (want & lowsel));
            if (fits) {
                cur.rsel = want;
            } else {
                segs.emplace_back();
                segs.back().rsel = tsel;
            }
        }
        flush(it.tmask, false);
        segs.back().ops.push_back(it.op);
    }
    if (carried) {
        carried->clear();
        for (size_t ii = 0; ii < pb.items.size(); ++ii) {
            const Item& it = pb.items[ii];
            if (!it.diag || touched[ii]) continue;
            bool out = false;
            for (const HTerm& t : it.terms) out |= (t.mask & ~W) != 0;
            if (out) {
                skip[ii] = 1;
                carried->push_back((int)ii);
            }
        }
    }
    flush(0, true);
    // the first and last segments touch HBM: their register bits must avoid the low bits
    if (segs.front().rsel & lowsel) segs.insert(segs.begin(), SegB());
    // a last segment whose registers hold low window bits stores in its own
    // layout: its lanes' window bits are written to the low physical bits
    // (coalesced) and the window bits are relabelled (TileSpec::operm, the
    // planner updates the qubit map) instead of one more SMEM transpose
    // Only the plan's final pass: a relabelled window changes which qubits sit
    // on the low bits for the passes after it (measured: QAOA30's later passes
    // lost more than the saved transposes, 44.0 -> 52.7 ms; QFT30's final pass
    // 6.22 -> 5.79 ms).  QJ_TILE_OPERM=0 off, =2 on every pass.
    static const char* operm_env = getenv("QJ_TILE_OPERM");
    const int operm_mode = operm_env ? atoi(operm_env) : 1;
    const bool operm = operm_mode > 0 && (final_pass || operm_mode == 2) && segs.size() > 1 && (segs.back().rsel & lowsel);
    if ((segs.back().rsel & lowsel) && !operm) segs.emplace_back();
    if ((int)segs.size() > TILE_MAXSEG) return false;
    // pad register sets to TILE_R bits (prefer high window bits)
    for (size_t s = 0; s < segs.size(); ++s) {
        const bool global = s == 0 || (s + 1 == segs.size() && !operm);
        for (int j = TILE_W - 1; j >= 0 && popc(segs[s].rsel) < TILE_R; --j) {
            if (global && ((lowsel >> j) & 1)) continue;
            segs[s].rsel |= 1u << j;
        }
    }
    for (size_t s = 0; s < segs.size(); ++s) {
        TSeg S;
        std::memset(&S, 0, sizeof(S));
        const bool global = s == 0 || (s + 1 == segs.size() && !operm);
        for (int j = 0, k = 0; j < TILE_W; ++j)
            if ((segs[s].rsel >> j) & 1) S.rbits[k++] = (int8_t)j;
        thread_bits(segs[s].rsel, C, M, global, S.tbits);
        S.op0 = (uint16_t)ts.ops.size();
        for (auto& op : segs[s].ops) ts.ops.push_back(op);
        S.op1 = (uint16_t)ts.ops.size();
        S.split = -1;
        ts.segs.push_back(S);
    }
    if (operm) {  // lanes 0..C-1 of the last segment -> window positions 0..C-1, the rest in order
        const TSeg& L = ts.segs.back();
        bool used[TILE_W] = {};
        for (int i = 0; i < C; ++i) {
            ts.operm[L.tbits[i]] = (int8_t)i;
            used[L.tbits[i]] = true;
        }
        for (int b = 0, pos = C; b < TILE_W; ++b)
            if (!used[b]) ts.operm[b] = (int8_t)pos++;
        ts.operm_on = true;
    }
    // Half-buffer transposes: the move into segment s can run
    // in two rounds through a buffer of 2^(W-1) amplitudes when one window bit
    // b sits at the same thread-id position p in both layouts -- round k is
    // done by the threads with tid bit p = k, which write and then read only
    // amplitudes with x_b = k.  b must lie above the swizzled low bits so the
    // compressed SMEM index keeps the bank mapping.  Segment s's order may be
    // permuted among its unconstrained positions (>= the lane constraint) to
    // line b up; segment s-1 is never touched, so earlier choices stay valid.
    const char* pipe = getenv("QJ_TILE_PIPE");  // only the pipelined JIT form uses splits
    for (size_t s = 1; s < ts.segs.size() && pipe && pipe[0] == '1'; ++s) {
        TSeg& P = ts.segs[s - 1];
        TSeg& S = ts.segs[s];
        const int lim = (s + 1 == ts.segs.size()) ? C : M;  // positions below are pinned
        int best = -1, bestq = -1;
        for (int p = TILE_T - 1; p >= 0 && best < 0; --p) {
            const int b = P.tbits[p];
            if (b < M) continue;  // swz<R> mixes the bits below M
            for (int q = 0; q < TILE_T; ++q)
                if (S.tbits[q] == b && (q == p || (q >= lim && p >= lim))) {
                    best = p;
                    bestq = q;
                    break;
                }
        }
        if (best < 0) continue;
        std::swap(S.tbits[best], S.tbits[bestq]);
        S.split = (int8_t)best;
    }
    return (int)ts.ops.size() <= TILE_MAXOPS;
}

void Planner::plan_fused(const PlanContext& ctx, const std::vector<LGate>& gates, std::vector<Step>& out) {
    if (ctx.nl < TILE_W + 2) {
        for (const LGate& g : gates) plan_gate(ctx, g, out);
        return;
    }
    std::vector<int>& phys = *ctx.phys;
    // 256-byte contiguous HBM runs (16 x c128 / 32 x c64): 128-byte runs cap a
    // pass with high window bits at ~0.66 of the HBM peak (tools/membench.cu)
    // with a 13-bit window; with 12 bits the window holds one fewer high bit
    // and 128-byte runs keep QFT30 at three passes
    int C = (ctx.amp_bytes == 16 ? 3 : 4) + (TILE_W >= 13 ? 1 : 0);
    const int M = ctx.amp_bytes == 16 ? 3 : 4;  // swizzle period (swz<R>): lanes of one SMEM wavefront
    if (const char* e = getenv("QJ_TILE_C")) {  // experiment: wider contiguous runs
        const int c = atoi(e);
        if (c >= 2 && c <= 6) C = c;
    }
    const uint64_t low = (1ull << C) - 1ull;
    const int max_terms = TILE_MAXTERMS;
    PassBuild pb;
    pb.W = low;
    // allow_carry: another pass follows, so diagonal terms still pending at the
    // end of this one may start it instead (build_tile)
    auto close = [&](bool allow_carry) {
        if (pb.items.empty()) return;
        PassBuild next;
        next.W = low;
        if (pb.singles.size() == 1) {
            // a single gate: the specialised single-gate pass touches fewer bytes
            for (const Step& st : pb.singles[0]) out.push_back(st);
        } else {
            Step s;
            s.type = Step::TILE;
            s.shard = 0;
            std::vector<int> carried;
            bool has_op = false;
            for (const Item& it : pb.items) has_op |= !it.diag;
            // opt-in (QJ_TILE_CARRY=1): measured slower -- the next pass's anchored runs
            // gain per-tile factors
            const bool carry = allow_carry && has_op && getenv("QJ_TILE_CARRY") && getenv("QJ_TILE_CARRY")[0] == '1';
            if (build_tile(pb, ctx.nl, C, M, s.tile, carry ? &carried : nullptr, !allow_carry) &&
                tile_fits(s.tile, ctx.nl, ctx.amp_bytes)) {
                for (int i : carried) {
                    next.nterms += (int)pb.items[i].terms.size();
                    next.cost += 0.05 * (double)pb.items[i].terms.size();
                    next.items.push_back(std::move(pb.items[i]));
                    next.singles.push_back(std::move(pb.singles[i]));
                }
                s.alg_bytes = 2.0 * ctx.amp_bytes * std::ldexp(1.0, ctx.nl);
                if (getenv("QJ_DEBUG_PLAN")) {
                    int nruns = 0, nterms = 0;
                    for (auto& op : s.tile.ops)
                        if (op.type == TO_RUN) {
                            ++nruns;
                            nterms += (int)op.terms.size();
                        }
                    fprintf(stderr, "[qj plan] tile pass: %zu gates, window", pb.singles.size());
                    for (int j = 0; j < TILE_W; ++j) fprintf(stderr, " %d", s.tile.wpos[j]);
                    fprintf(stderr, " | %zu segs, %zu ops, %d runs, %d terms\n", s.tile.segs.size(),
                            s.tile.ops.size(), nruns, nterms);
                    if (getenv("QJ_DEBUG_PLAN")[0] == '2')
                        for (const TSeg& S : s.tile.segs) {
                            fprintf(stderr, "    seg r:");
                            for (int j = 0; j < TILE_R; ++j) fprintf(stderr, " %d", S.rbits[j]);
                            fprintf(stderr, " t:");
                            for (int j = 0; j < TILE_T; ++j) fprintf(stderr, " %d", S.tbits[j]);
                            fprintf(stderr, " split %d\n", S.split);
                        }
                }
                // one pass per shard: the same program, the shard's global bits
                // enter the predicates through gbase (tile.h)
                for (int r = 0; r < ctx.nshards; ++r) {
                    Step sr = s;
                    sr.shard = r;
                    sr.tile.gbase = (uint64_t)r << ctx.nl;
                    out.push_back(std::move(sr));
                }
                if (s.tile.operm_on) {  // the pass wrote window bit b at window position operm[b]
                    int where[64];
                    for (int b = 0; b < 64; ++b) where[b] = b;
                    for (int b = 0; b < TILE_W; ++b) where[s.tile.wpos[b]] = s.tile.wpos[s.tile.operm[b]];
                    for (int& p : phys)
                        if (p < 64) p = where[p];
                }
            } else {
                // cannot happen with the limits below; stay correct anyway
                for (const auto& v : pb.singles)
                    for (const Step& st : v) out.push_back(st);
            }
        }
        pb = std::move(next);
    };
    auto single = [&](const LGate& g) {
        std::vector<Step> v;
        for (int r = 0; r < ctx.nshards; ++r) {
            Step s;
            s.type = Step::PASS;
            s.shard = r;
            if (!specialise(ctx, g, (uint64_t)r, s.pass)) continue;  // identity on this shard
            s.alg_bytes = pass_alg_bytes(s.pass, ctx.nl, ctx.amp_bytes);
            v.push_back(std::move(s));
        }
        return v;
    };
    // DAG-aware packing: a gate that does not fit the current pass is deferred
    // and blocks its qubits; later gates that depend on no deferred gate keep
    // joining the pass (they commute with everything deferred).  Deferred
    // gates start the next pass, in program order.
    std::vector<int> remaining(gates.size());
    for (size_t i = 0; i < gates.size(); ++i) remaining[i] = (int)i;
    std::vector<char> blocked(ctx.n, 0);
    // arithmetic per amplitude a pass may take before it closes (cost units of
    // op_cost); swept on B200 with the zero-pattern cost model (round 2): c64
    // sup32 915 -> 800 / 762 ms at 128 / 192; c128 stays at 96 -- at 128 QAOA30
    // gains 44.9 -> 43.0 ms but BV30's pre-fused plan wins the byte comparison
    // with a compute-heavy pass (8.7 -> 18.4 ms)
    double budget = ctx.amp_bytes == 16 ? 96.0 : 192.0;
    if (const char* b = getenv("QJ_TILE_BUDGET")) budget = atof(b);
    const bool dag = !(getenv("QJ_TILE_DAG") && getenv("QJ_TILE_DAG")[0] == '0');
    while (!remaining.empty()) {
        std::vector<int> deferred;
        std::fill(blocked.begin(), blocked.end(), 0);
        auto defer = [&](int idx) {
            deferred.push_back(idx);
            const LGate& g = gates[idx];
            for (int i = 0; i < g.nt; ++i) blocked[g.t[i]] = 1;
            for (int i = 0; i < g.nc; ++i) blocked[g.c[i]] = 1;
        };
        for (int idx : remaining) {
            const LGate& g = gates[idx];
            bool blk = false;
            for (int i = 0; i < g.nt; ++i) blk |= blocked[g.t[i]] != 0;
            for (int i = 0; i < g.nc; ++i) blk |= blocked[g.c[i]] != 0;
            if (blk) {
                defer(idx);
                continue;
            }
            if (g.kind == QJ_GATE_SWAP && g.nc == 0) {
                // relabel: the two logical qubits exchange physical bits
                std::swap(phys[g.t[0]], phys[g.t[1]]);
                continue;
            }
            Item it;
            std::vector<HTerm> terms;
            if (diag_terms(g, phys, terms)) {
                if (pb.nterms + (int)terms.size() > max_terms - 8 || pb.cost + 0.05 > budget) {
                    defer(idx);
                    continue;
                }
                it.diag = true;
                it.terms = std::move(terms);
                pb.nterms += (int)it.terms.size();
                pb.cost += 0.05 * (double)it.terms.size();
                pb.items.push_back(std::move(it));
                pb.singles.push_back(single(g));
                continue;
            }
            if (needs_exchange(ctx, g)) {
                // a global target: swap it into the local bits between passes
                if (pb.items.empty() && deferred.empty()) {
                    exchange_for(ctx, g, out);
                } else {
                    defer(idx);
                    continue;
                }
            }
            HOp op;
            if (!make_op(g, phys, op)) {
                // not fusable: runs alone once nothing earlier is pending
                if (pb.items.empty() && deferred.empty()) {
                    plan_gate(ctx, g, out);
                } else {
                    defer(idx);
                }
                continue;
            }
            uint64_t tm = 0;
            for (int i = 0; i < g.nt; ++i) tm |= 1ull << op.t[i];
            const int nm = (int)op.m.size();
            const double c = op_cost(op);
            const bool fits = popc(pb.W | tm) <= TILE_W && pb.nops + 2 <= kMaxOpsPerPass &&
                              pb.nmat + nm <= kMaxMatPerPass && pb.nnd + 1 < TILE_MAXRUNS &&
                              (pb.cost + c <= budget || pb.items.empty());
            if (!fits) {
                defer(idx);
                if (!dag) {  // sequential packing: everything after waits for the next pass
                    for (int q = 0; q < ctx.n; ++q) blocked[q] = 1;
                }
                continue;
            }
            pb.cost += c;
            pb.W |= tm;
            pb.nops += 2;  // the op plus a possible run flush before it
            pb.nnd += 1;
            pb.nmat += nm;
            it.op = std::move(op);
            it.tmask = tm;
            pb.items.push_back(std::move(it));
            pb.singles.push_back(single(g));
        }
        close(!deferred.empty());
        remaining.swap(deferred);
    }
    close(false);  // terms carried out of the last pass
}

}  // namespace qj
