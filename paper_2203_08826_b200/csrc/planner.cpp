// planner.cpp -- see planner.h.
#include "planner.h"
#include "small.h"

#include <cstdlib>

#include <algorithm>
#include <cmath>

namespace qj {

double pass_alg_bytes(const Pass& p, int nl, int amp_bytes) {
    double touched = std::ldexp(1.0, nl - p.nfix);
    switch (p.kind) {
        case PK_DENSE: {
            const int D = 1 << p.k;
            const uint32_t m = D >= 32 ? 0xffffffffu : ((1u << D) - 1u);
            touched *= (double)__builtin_popcount(p.touch & m) / (double)D;
            break;
        }
        case PK_SWAP: touched *= 0.5; break;
        default: break;
    }
    return 2.0 * amp_bytes * touched;
}

static bool is_diagonal(const std::vector<cd>& m, int D) {
    for (int r = 0; r < D; ++r)
        for (int c = 0; c < D; ++c)
            if (r != c && m[(size_t)r * D + c] != cd(0, 0)) return false;
    return true;
}

bool specialise(const PlanContext& ctx, const LGate& g, uint64_t r, Pass& p) {
    const std::vector<int>& phys = *ctx.phys;
    const int nl = ctx.nl;
    p = Pass();
    // controls: local -> fixed bit = 1; global -> shard filter
    for (int i = 0; i < g.nc; ++i) {
        const int b = phys[g.c[i]];
        if (b >= nl) {
            if (!((r >> (b - nl)) & 1u)) return false;
        } else {
            p.fpos[p.nfix] = b;
            p.fval[p.nfix++] = 1;
        }
    }
    int kind = g.kind;
    std::vector<cd> diag;
    if (kind == QJ_GATE_DENSE) {
        const int D = 1 << g.nt;
        if (is_diagonal(g.data, D)) {
            kind = QJ_GATE_DIAG;
            diag.resize(D);
            for (int i = 0; i < D; ++i) diag[i] = g.data[(size_t)i * D + i];
        }
    } else if (kind == QJ_GATE_DIAG) {
        diag = g.data;
    } else if (kind == QJ_GATE_Z) {
        kind = QJ_GATE_DIAG;
        diag = {cd(1, 0), cd(-1, 0)};
    }
    if (kind == QJ_GATE_DIAG) {
        // slice global target bits by shard r
        int lt[QJ_MAX_TARGETS], lidx[QJ_MAX_TARGETS], nlt = 0;
        uint32_t gfixed = 0;  // bits of the full row index fixed by r
        for (int i = 0; i < g.nt; ++i) {
            const int b = phys[g.t[i]];
            if (b >= nl) {
                if ((r >> (b - nl)) & 1u) gfixed |= 1u << (g.nt - 1 - i);
            } else {
                lt[nlt] = b;
                lidx[nlt++] = i;
            }
        }
        std::vector<cd> loc((size_t)1 << nlt);
        for (int lr = 0; lr < (1 << nlt); ++lr) {
            uint32_t full = gfixed;
            for (int j = 0; j < nlt; ++j)
                if ((lr >> (nlt - 1 - j)) & 1) full |= 1u << (g.nt - 1 - lidx[j]);
            loc[lr] = diag[full];
        }
        int nonunit = 0, which = -1;
        for (int i = 0; i < (int)loc.size(); ++i)
            if (loc[i] != cd(1, 0)) {
                ++nonunit;
                which = i;
            }
        if (nonunit == 0) return false;  // identity on this shard
        if (nonunit == 1) {
            // phase on the subspace where the local target bits spell `which`
            for (int j = 0; j < nlt; ++j) {
                p.fpos[p.nfix] = lt[j];
                p.fval[p.nfix++] = (which >> (nlt - 1 - j)) & 1;
            }
            if (loc[which] == cd(-1, 0)) {
                p.kind = PK_NEG;
            } else {
                p.kind = PK_PHASE;
                p.m = {loc[which]};
            }
            return true;
        }
        p.kind = PK_DIAG;
        p.k = nlt;
        for (int j = 0; j < nlt; ++j) p.tpos[j] = lt[j];
        p.m = loc;
        return true;
    }
    // non-diagonal: all targets are local here (remapped by the planner)
    p.k = g.nt;
    for (int i = 0; i < g.nt; ++i) p.tpos[i] = phys[g.t[i]];
    switch (kind) {
        case QJ_GATE_X: p.kind = PK_X; break;
        case QJ_GATE_SWAP: p.kind = PK_SWAP; break;
        case QJ_GATE_FSIM: {
            p.kind = PK_DENSE;
            p.m.assign(16, cd(0, 0));
            p.m[0] = 1;
            p.m[5] = g.data[0];
            p.m[6] = g.data[1];
            p.m[9] = g.data[2];
            p.m[10] = g.data[3];
            p.m[15] = g.data[4];
            p.touch = 0xEu;  // members 01, 10, 11
            break;
        }
        default:
            p.kind = PK_DENSE;
            p.m = g.data;
            break;
    }
    return true;
}

static bool nondiagonal(const LGate& g) {
    switch (g.kind) {
        case QJ_GATE_X:
        case QJ_GATE_SWAP:
        case QJ_GATE_FSIM:
            return true;
        case QJ_GATE_DENSE:
            return !is_diagonal(g.data, 1 << g.nt);
        default:
            return false;
    }
}

bool needs_exchange(const PlanContext& ctx, const LGate& g) {
    if (ctx.g == 0 || !nondiagonal(g)) return false;
    for (int i = 0; i < g.nt; ++i)
        if ((*ctx.phys)[g.t[i]] >= ctx.nl) return true;
    return false;
}

// Bring every global target of a non-diagonal gate into the local bits:
// EXCHANGE with the highest local bit the gate does not use; updates the map.
void exchange_for(const PlanContext& ctx, const LGate& g, std::vector<Step>& out) {
    std::vector<int>& phys = *ctx.phys;
    if (!needs_exchange(ctx, g)) return;
    for (int i = 0; i < g.nt; ++i) {
        const int b = phys[g.t[i]];
        if (b < ctx.nl) continue;
        int L = -1;
        for (int cand = ctx.nl - 1; cand >= 0 && L < 0; --cand) {
            bool used = false;
            for (int j = 0; j < g.nt; ++j) used |= phys[g.t[j]] == cand;
            for (int j = 0; j < g.nc; ++j) used |= phys[g.c[j]] == cand;
            if (!used) L = cand;
        }
        Step s;
        s.type = Step::EXCHANGE;
        s.gbit = b - ctx.nl;
        s.lbit = L;
        out.push_back(s);
        for (int q = 0; q < ctx.n; ++q) {
            if (phys[q] == b) phys[q] = L;
            else if (phys[q] == L) phys[q] = b;
        }
    }
}

void Planner::plan_gate(const PlanContext& ctx, const LGate& g, std::vector<Step>& out) {
    exchange_for(ctx, g, out);
    for (int r = 0; r < ctx.nshards; ++r) {
        Step s;
        s.type = Step::PASS;
        s.shard = r;
        if (!specialise(ctx, g, (uint64_t)r, s.pass)) continue;
        s.alg_bytes = pass_alg_bytes(s.pass, ctx.nl, ctx.amp_bytes);
        out.push_back(std::move(s));
    }
}

// States that fit one SM's shared memory run whole runs of gates in ONE
// launch of the SMEM kernel (small.h); passes it does not take (dense k > 4)
// run as ordinary passes in between.
static bool small_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("QJ_SMALL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// QJ_AUTO_FUSE=0 disables the automatic choice of pre-fused tile plans.
static bool auto_fuse_enabled() {
    static const bool on = !(getenv("QJ_AUTO_FUSE") && getenv("QJ_AUTO_FUSE")[0] == '0');
    return on;
}

void Planner::plan(const PlanContext& ctx, const std::vector<LGate>& gates, bool fuse, std::vector<Step>& out) {
    if (fuse && ctx.nshards == 1 && ctx.n <= small_max_qubits(ctx.amp_bytes) && small_enabled()) {
        std::vector<Step> tmp;
        Step cur;
        cur.type = Step::SMALL;
        const double bytes = 2.0 * ctx.amp_bytes * (double)(1ull << ctx.nl);
        auto flush = [&]() {
            if (cur.prog.empty()) return;
            cur.alg_bytes = bytes;
            out.push_back(std::move(cur));
            cur = Step();
            cur.type = Step::SMALL;
        };
        for (const LGate& g : gates) {
            tmp.clear();
            plan_gate(ctx, g, tmp);
            for (Step& st : tmp) {
                if (st.type == Step::PASS && small_supports(st.pass)) {
                    cur.prog.push_back(std::move(st.pass));
                } else {
                    flush();
                    out.push_back(std::move(st));
                }
            }
        }
        flush();
        return;
    }
    if (fuse && auto_fuse_ && auto_fuse_enabled()) {
        // Window tile passes after the paper's <= 2-qubit gate fusion, or on
        // the gates as given: keep the plan that moves fewer algorithmic HBM
        // bytes (dense fused 4x4 matrices absorb 1q gates into their 2q
        // neighbours -- fewer ops per pass for random circuits -- but turn
        // diagonal phases into dense work, which QFT-like circuits lose on).
        std::vector<int> phys_a = *ctx.phys, phys_b = *ctx.phys;
        PlanContext ca = ctx, cb = ctx;
        ca.phys = &phys_a;
        cb.phys = &phys_b;
        std::vector<Step> a, b;
        plan_fused(ca, gates, a);
        plan_fused(cb, fuse_gates(gates, ctx.n, 2), b);
        auto bytes = [](const std::vector<Step>& v) {
            double t = 0;
            for (const Step& st : v) t += st.alg_bytes;
            return t;
        };
        const bool take_b = bytes(b) < 0.9 * bytes(a);
        *ctx.phys = take_b ? phys_b : phys_a;
        for (Step& st : take_b ? b : a) out.push_back(std::move(st));
        return;
    }
    if (fuse) {
        plan_fused(ctx, gates, out);
        return;
    }
    for (const LGate& g : gates) plan_gate(ctx, g, out);
}

}  // namespace qj
