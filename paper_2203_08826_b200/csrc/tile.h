// tile.h -- the fused window tile pass: one HBM round trip applies a run of
// consecutive gates whose non-diagonal targets lie in a window of TILE_W bits
// (the B200 form of the paper's "fewer state passes" gate
// fusion).
//
// Tile: the 2^TILE_W amplitudes sharing all non-window bits.  A block of
// TILE_THREADS threads owns one tile at a time; each thread holds TILE_NREG =
// 2^TILE_R amplitudes in registers.  The gate list of a pass is split into
// SEGMENTS; in segment s the register index bits map to 4 window bits R_s and
// the thread index bits to the other 8.  Gates on R_s run in registers;
// moving to the next segment transposes through XOR-swizzled shared memory.
// The first segment loads from HBM and the last stores to HBM directly
// (lanes 0..C-1 on the low window bits: 128-byte contiguous runs).
//
// Diagonal gates never need their bits in R: they are decomposed into phase
// TERMS (mask/value/factor over <= 3 bits) that commute with every gate not
// targeting their bits, deferred, and applied in merged RUNS.  Terms are
// classified per segment by where their bits live (C = outside the window,
// T = thread bits, R = register bits):
//   SLOT runs:   S  (C bits only), CT (one T bit + C), CR (one R bit + C):
//                products per tile (computed once per tile into SMEM), applied
//                as a thread scalar and per-register-bit factor pairs;
//   ANCHORED runs: terms that all contain one window bit b (the anchor) and at
//                most one other bit a: the factor on amplitudes with x_b = v is
//                slot(tile) * prod_a g[v][a][x_a]; the g tables are
//                tile-independent (computed on the host);
//   GENERIC L terms (anything else) are evaluated per thread.
// The bulky tables live in a device program buffer (TileTables) filled per
// pass through a pinned staging ring; the kernel parameters hold the
// geometry, ops and run descriptors.
#pragma once

#include <stdint.h>

#include <vector>

#include "common.cuh"
#include "qj_internal.h"

namespace qj {

constexpr int TILE_W = 12;
constexpr int TILE_R = 4;
constexpr int TILE_T = TILE_W - TILE_R;  // 8 thread bits
constexpr int TILE_THREADS = 1 << TILE_T;
constexpr int TILE_NREG = 1 << TILE_R;
constexpr int TILE_MAXSEG = 8;
constexpr int TILE_MAXOPS = 160;
constexpr int TILE_MAXCX = 64;
constexpr int TILE_MAXRUNS = 96;
constexpr int TILE_MAXSLOTS = 1024;
constexpr int TILE_MAXTERMS = 1024;  // planner budget per pass
constexpr int TILE_MAXMAT = 1024;    // complex entries in the matrix pool

enum TOpType : uint8_t {
    TO_H = 0,     // Hadamard on R bit a
    TO_U1 = 1,    // 2x2 matrix (mat) on R bit a
    TO_U2 = 2,    // 4x4 matrix (mat) on R bits (a = MSB, b)
    TO_X = 3,     // X on R bit a
    TO_SWAP = 4,  // SWAP R bits a, b
    TO_RUN = 5,   // phase run `run`
};

struct TOp {
    uint8_t type, a, b;
    uint8_t cr_mask, cr_val;  // controls on R bits (R-local bit mask / value)
    uint8_t pad0;
    uint16_t idx;             // matrix offset (U1/U2) or run index (RUN)
    int16_t cx;               // index into cx[] (controls on non-R bits), -1 = none
    uint16_t pad1[3];
};

struct TSeg {
    int8_t tbits[TILE_T];  // window-bit index mapped to thread-id bit i
    int8_t rbits[TILE_R];  // window-bit index mapped to register-index bit j
    uint16_t op0, op1;     // op range
};

enum TRunKind : uint8_t { RUN_SLOT = 0, RUN_ANCHOR = 1 };

struct TRunDesc {
    uint8_t kind;
    // ---- RUN_SLOT
    uint8_t ru;          // register bits with CR slots / single-R-bit L terms
    uint8_t r0one;       // register bits whose value-0 factor is always 1
    uint8_t has_scalar;  // S / CT / L-scalar contributions exist
    int16_t s_slot;
    int16_t ct_slot[TILE_T][2];
    int16_t cr_slot[TILE_R][2];
    uint16_t l0, l1;  // generic L term range
    int32_t ta;       // per-thread scalar table (256 complex) offset in fac, -1 none
    int32_t tb;       // per-thread register-bit pairs (256 x 4 x 2 complex) offset in fac, -1 none
    int32_t pt;       // uniform register-pattern table (16 complex) offset in fac, -1 none
    // ---- RUN_ANCHOR
    uint8_t anc_r;     // 1: anchor is register bit anc, 0: thread bit anc
    uint8_t anc;
    uint8_t vmask;     // values of the anchor with terms (bit v)
    uint8_t tm[2];     // per v: thread bits with factors
    uint8_t rm[2];     // per v: register bits with factors
    uint8_t r1only[2]; // per v: register bits whose x=0 factor is 1
    int16_t aslot[2];  // per v: per-tile slot (C partner bits and anchor-only terms), -1 none
    uint32_t fac;      // offset of the factor table: [v][T bit][x] (32) then [v][R bit][x] (16)
    int32_t ft;        // per-thread thread-partner products [v][tid] offset in fac, -1 none
};

template <typename R>
struct TTerm {
    uint64_t cmask, cval;  // predicate over non-R physical bits (L) or C bits (slots)
    uint8_t rmask, rval;   // R-local pattern (L terms)
    uint8_t pad[6];
    Cx<R> f;
};

struct TSlot {
    uint32_t t0, t1;  // term range whose product (with tile predicate) fills the slot
};

// Device program buffer layout of one pass (offsets in bytes from the base).
struct TileTablesLayout {
    uint32_t terms, slots, mats, fac;
};

template <typename R>
struct TileArgs {
    void* psi;
    const unsigned char* tables;  // device program buffer of this pass
    TileTablesLayout lay;
    uint64_t ntiles;
    int nseg, nops, nslots, pad;
    int wpos[TILE_W];  // ascending physical positions of the window bits
    TSeg seg[TILE_MAXSEG];
    uint64_t tph[TILE_MAXSEG][2][16];  // physical offset of thread-id nibbles per segment
    uint32_t tlo[TILE_MAXSEG][2][16];  // window-local offset of thread-id nibbles
    TOp ops[TILE_MAXOPS];
    uint64_t cx[TILE_MAXCX][2];
    TRunDesc runs[TILE_MAXRUNS];
};

// Host-side description of one planned tile pass (precision-independent).
struct HTerm {
    uint64_t mask = 0, val = 0;  // physical bits / values of the pattern
    cd f;
};
struct HOp {
    int type = TO_U1;
    int t[2] = {0, 0};          // physical target bits (t[0] = matrix MSB)
    uint64_t cmask = 0;         // physical control bits (all 1)
    std::vector<cd> m;          // U1: 4, U2: 16
    std::vector<HTerm> terms;   // RUN
};
struct TileSpec {
    int w = 0;
    int wpos[TILE_W] = {};
    std::vector<TSeg> segs;
    std::vector<HOp> ops;        // ops in order; segs[].op0/op1 index into it
};

// Pinned-host + device ring for the per-pass program buffers.
struct TileStaging {
    static constexpr int kSlots = 8;
    static constexpr size_t kBytes = 256 * 1024;
    unsigned char* host = nullptr;  // pinned, kSlots * kBytes
    unsigned char* dev = nullptr;   // device, kSlots * kBytes
    cudaEvent_t ev[kSlots] = {};
    int next = 0;
    cudaError_t init();
    void release();
};

template <typename R>
cudaError_t run_tile(const TileSpec& t, void* psi, int nl, cudaStream_t st, TileStaging& stg, LaunchStats& ls);

// Whether a planned pass lowers within the kernel's capacities.
bool tile_fits(const TileSpec& t, int nl, int amp_bytes);

}  // namespace qj
