// tile_pass.cu -- the fused window tile pass kernel (see tile.h) and its
// launcher, which lowers a host TileSpec into the kernel's parameter block
// plus a device program buffer (terms, slots, matrices, anchored factors).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>

#include "tile.h"
#include "tile_dev.cuh"
#include "tile_jit.h"

namespace qj {

// the JIT kernels take TileArgs by value through cuLaunchKernel (4 KiB..32 KiB parameter space)
static_assert(sizeof(TileArgs<double>) <= 32764 && sizeof(TileArgs<float>) <= 32764, "TileArgs exceeds the kernel parameter limit");


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
    a->ntiles = 1ull << (nl - TILE_W - __builtin_popcountll(t.fix_mask));
    a->namps = 1ull << nl;
    a->chk = tile_check_flag();
    a->gbase = t.gbase;
    a->synth = t.synth_index;
    a->fixmask = t.fix_mask;
    a->fixval = t.fix_val & t.fix_mask;
    a->zmask = t.zero_mask;
    a->zval = t.zero_val & t.zero_mask;
    a->bins = t.bins;
    a->nbq = t.nbins_q;
    a->fflags = (t.synth ? 1 : 0) | (t.nbins_q > 0 ? 2 : 0);
    for (int k = 0; k < t.nbins_q; ++k) a->bin_pos[k] = t.bin_pos[k];
    // output positions of window bits (identity unless the last segment stores in its own layout)
    a->has_operm = t.operm_on ? 1 : 0;
    int opos[TILE_W];
    for (int b = 0; b < TILE_W; ++b) {
        a->operm[b] = (int8_t)(t.operm_on ? t.operm[b] : b);
        opos[b] = t.wpos[a->operm[b]];
    }
    {
        const TSeg& S = t.segs.back();
        for (int half = 0; half < TILE_TCH; ++half)
            for (int nib = 0; nib < 16; ++nib) {
                uint64_t ph = 0;
                for (int q = 0; q < 4; ++q)
                    if (((nib >> q) & 1) && half * 4 + q < TILE_T) ph |= 1ull << opos[S.tbits[half * 4 + q]];
                a->tph_out[half][nib] = ph;
            }
    }
    if (t.nbins_q > 0) {  // register-index part of the bin for the last segment's (output) mapping
        const TSeg& S = t.segs.back();
        for (int r = 0; r < TILE_NREG; ++r) {
            uint64_t x = 0;
            for (int j = 0; j < TILE_R; ++j)
                if ((r >> j) & 1) x |= 1ull << opos[S.rbits[j]];
            uint32_t b = 0;
            for (int k = 0; k < t.nbins_q; ++k) b = (b << 1) | (uint32_t)((x >> t.bin_pos[k]) & 1u);
            a->regbin[r] = (uint16_t)b;
        }
    }
    a->nseg = (int)t.segs.size();
    a->nops = (int)t.ops.size();
    uint64_t wmask = 0;
    for (int i = 0; i < TILE_W; ++i) {
        a->wpos[i] = t.wpos[i];
        wmask |= 1ull << t.wpos[i];
    }
    if (t.zero_mask & ~wmask) return false;
    if (t.fix_mask & (wmask | ~((nl >= 64 ? 0ull : 1ull << nl) - 1))) return false;  // fixed bits: local, outside W
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
        for (int half = 0; half < TILE_TCH; ++half)
            for (int nib = 0; nib < 16; ++nib) {
                uint64_t ph = 0;
                uint32_t lo = 0;
                for (int q = 0; q < 4; ++q)
                    if (((nib >> q) & 1) && half * 4 + q < TILE_T) {
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
            // slot terms on an anchor bit (the anchor plus at most one C bit) join that
            // anchored run: its per-tile slot factor folds into the run's scalar
            // instead of a second multiply of the same registers
            if (!groups.empty()) {
                std::vector<const HTerm*> keep;
                for (auto* ht : slotable) {
                    const uint64_t wb = ht->mask & wmask;
                    int gi = -1;
                    if (wb && popc64(wb) == 1 && popc64(ht->mask) <= 2)
                        for (size_t q = 0; q < groups.size(); ++q)
                            if (wb == (1ull << groups[q].first)) gi = (int)q;
                    if (gi >= 0) groups[gi].second.push_back(ht);
                    else keep.push_back(ht);
                }
                slotable.swap(keep);
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
    // tile + two slot tables (the JIT kernel double-buffers them across tiles)
    const size_t smem = sizeof(Cx<R>) * ((size_t)(1 << TILE_W) + 2 * (size_t)std::max(a->nslots, 1));
    static size_t attr = 0;
    if (smem > attr) {
        const size_t want = sizeof(Cx<R>) * ((size_t)(1 << TILE_W) + 2 * TILE_MAXSLOTS);
        e = cudaFuncSetAttribute(tile_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
        if (e != cudaSuccess) return e;
        attr = want;
    }
    const int sms = device_sms();
    const uint64_t grid = std::min<uint64_t>(a->ntiles, (uint64_t)sms * TILE_MINBLOCKS);
    std::string jerr;
    const JitKernel* jk = tile_jit_kernel<R>(*a, blob.empty() ? nullptr : blob.data(), &jerr, nullptr);
    if (jk) {
        tile_jit_fill<R>(*jk, a, blob.data());
        if (jk->tmap) {
            e = tile_jit_encode_tmap<R>(a, jk->l2_256);
            if (e != cudaSuccess) return e;
        }
        const uint64_t jgrid = std::min<uint64_t>(a->ntiles, (uint64_t)sms * jk->blocks);
        e = tile_jit_launch(jk->f, a, (unsigned)jgrid, smem + jk->smem_extra, st, jk->threads);
    } else {
        static bool warned = false;
        if (!warned && getenv("QJ_DEBUG_JIT")) fprintf(stderr, "[qj jit] interpreter fallback: %s\n", jerr.c_str());
        warned = true;
        tile_kernel<R><<<(unsigned)grid, TILE_THREADS, smem, st>>>(*a);
        e = cudaGetLastError();
    }
    ls.launches++;
    return e;
}

template <typename R>
cudaError_t tile_prepare(const TileSpec& t, void* psi, int nl, PreparedTile& out) {
    static TileArgs<R>* a = new TileArgs<R>;
    std::vector<unsigned char> blob;
    if (!lower_tile<R>(t, nl, a, blob)) return cudaErrorInvalidValue;
    a->psi = psi;
    out.amp_bytes = (int)(2 * sizeof(R));
    if (!blob.empty()) {
        cudaError_t e = cudaMalloc(&out.dev, blob.size());
        if (e != cudaSuccess) return e;
        e = cudaMemcpy(out.dev, blob.data(), blob.size(), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return e;
    }
    a->tables = static_cast<const unsigned char*>(out.dev);
    out.smem = sizeof(Cx<R>) * ((size_t)(1 << TILE_W) + 2 * (size_t)std::max(a->nslots, 1));
    static size_t attr = 0;
    if (out.smem > attr) {
        const size_t want = sizeof(Cx<R>) * ((size_t)(1 << TILE_W) + 2 * TILE_MAXSLOTS);
        cudaError_t e = cudaFuncSetAttribute(tile_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)want);
        if (e != cudaSuccess) return e;
        attr = want;
    }
    const int sms = device_sms();
    out.grid = (unsigned)std::min<uint64_t>(a->ntiles, (uint64_t)sms * TILE_MINBLOCKS);
    std::string jerr;
    const JitKernel* jk = tile_jit_kernel<R>(*a, blob.empty() ? nullptr : blob.data(), &jerr, nullptr);
    out.jit = jk ? jk->f : nullptr;
    if (jk) {
        tile_jit_fill<R>(*jk, a, blob.data());
        if (jk->tmap) {
            cudaError_t e = tile_jit_encode_tmap<R>(a, jk->l2_256);
            if (e != cudaSuccess) return e;
        }
        out.smem += jk->smem_extra;
        out.grid = (unsigned)std::min<uint64_t>(a->ntiles, (uint64_t)sms * jk->blocks);
        out.threads = jk->threads;
    }
    out.args.assign(reinterpret_cast<unsigned char*>(a), reinterpret_cast<unsigned char*>(a) + sizeof(TileArgs<R>));
    return cudaSuccess;
}

cudaError_t tile_launch_prepared(const PreparedTile& p, cudaStream_t st, LaunchStats& ls) {
    cudaError_t e;
    if (p.jit) {
        e = tile_jit_launch(p.jit, p.args.data(), p.grid, p.smem, st, p.threads);
    } else if (p.amp_bytes == 16) {
        tile_kernel<double><<<p.grid, TILE_THREADS, p.smem, st>>>(*reinterpret_cast<const TileArgs<double>*>(p.args.data()));
        e = cudaGetLastError();
    } else {
        tile_kernel<float><<<p.grid, TILE_THREADS, p.smem, st>>>(*reinterpret_cast<const TileArgs<float>*>(p.args.data()));
        e = cudaGetLastError();
    }
    ls.launches++;
    return e;
}

void tile_release(PreparedTile& p) {
    if (p.dev) cudaFree(p.dev);
    p.dev = nullptr;
}

template bool lower_tile<float>(const TileSpec&, int, TileArgs<float>*, std::vector<unsigned char>&);
template bool lower_tile<double>(const TileSpec&, int, TileArgs<double>*, std::vector<unsigned char>&);
template cudaError_t tile_prepare<float>(const TileSpec&, void*, int, PreparedTile&);
template cudaError_t tile_prepare<double>(const TileSpec&, void*, int, PreparedTile&);
template cudaError_t run_tile<float>(const TileSpec&, void*, int, cudaStream_t, TileStaging&, LaunchStats&);
template cudaError_t run_tile<double>(const TileSpec&, void*, int, cudaStream_t, TileStaging&, LaunchStats&);

}  // namespace qj
