// tile_abi.h -- parameter / program-buffer layout shared by the host lowering
// (tile_pass.cu), the ahead-of-time interpreter kernel and the run-time
// compiled (NVRTC) tile kernels (tile_jit.cpp).  Plain PODs only: this header
// is also compiled by NVRTC.
#pragma once

#include "common.cuh"

namespace qj {

#ifndef QJ_TILE_R
#define QJ_TILE_R 4
#endif
#ifndef QJ_TILE_W
#define QJ_TILE_W 12
#endif
constexpr int TILE_W = QJ_TILE_W;            // window bits: a tile is 2^TILE_W amplitudes
constexpr int TILE_R = QJ_TILE_R;          // register bits per thread (3 or 4)
constexpr int TILE_T = TILE_W - TILE_R;    // thread-index bits
constexpr int TILE_THREADS = 1 << TILE_T;
constexpr int TILE_NREG = 1 << TILE_R;
constexpr int TILE_TCH = (TILE_T + 3) / 4;  // 4-bit chunks of the thread index
#ifndef QJ_TILE_MINBLOCKS
#define QJ_TILE_MINBLOCKS (QJ_TILE_W >= 13 ? 1 : 2)
#endif
constexpr int TILE_MINBLOCKS = QJ_TILE_MINBLOCKS;  // resident CTAs per SM (JIT kernels: per-launch option)
constexpr int TILE_MAXSEG = 8;
constexpr int TILE_MAXOPS = 160;
constexpr int TILE_MAXCX = 64;
constexpr int TILE_MAXRUNS = 96;
constexpr int TILE_MAXSLOTS = 1024;
constexpr int TILE_MAXTERMS = 1024;  // planner budget per pass
constexpr int TILE_MAXMAT = 1024;    // complex entries in the matrix pool
constexpr int TILE_MAXUC = 512;     // uniform coefficients staged in the kernel-parameter block (JIT)

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
    int8_t split;          // thread-id bit that holds the same window bit in this and the
                           // previous segment (half-buffer transposes), -1 = none
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
    int16_t cr_slot[4][2];
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

// Ring form (JIT): the tile as a TMA box of a <= 5-D view of the state
// (doubles; dim 0 = the window's low contiguous bits x amplitude, then
// alternating window segments (box = extent, <= 256) and gap segments (box 1,
// the tile's coordinate)); smem receives the tile in window-local order.
struct TmapGeom {
    int rank = 0;
    uint64_t extent[5] = {};
    uint64_t stride_bytes[5] = {};  // [0] unused (contiguous)
    uint32_t box[5] = {};
    int start_bit[5] = {};          // amplitude-index bit where the dim starts
    int len[5] = {};                // its bits (dim 0: amplitude bits only)
    bool gap[5] = {};
};

template <typename R>
struct TileArgs {
    alignas(64) unsigned char tmap[128];  // CUtensorMap of the ring form's TMA loads (JIT ring kernels only)
    void* psi;
    const unsigned char* tables;  // device program buffer of this pass
    TileTablesLayout lay;
    uint64_t ntiles;
    uint64_t gbase;  // global-bit part of the physical index (sharded states); predicates only
    int nseg, nops, nslots, pad;
    int wpos[TILE_W];  // ascending physical positions of the window bits
    TSeg seg[TILE_MAXSEG];
    uint64_t tph[TILE_MAXSEG][TILE_TCH][16];  // physical offset of thread-id nibbles per segment
    uint32_t tlo[TILE_MAXSEG][TILE_TCH][16];  // window-local offset of thread-id nibbles
    TOp ops[TILE_MAXOPS];
    uint64_t cx[TILE_MAXCX][2];
    TRunDesc runs[TILE_MAXRUNS];
    // JIT kernels: tile-independent uniform coefficients (gate matrices, anchored
    // phase factors, pattern tables) copied here at launch, so they are read
    // through the constant bank instead of per-tile global loads
    Cx<R> uc[TILE_MAXUC];
    // qj_simulate fusions (JIT kernels; see tile.h)
    uint64_t synth;          // local index of the basis amplitude (synthesised first pass)
    uint64_t fixval;         // live-tile passes: value of the fixed bits (fixmask), OR-ed into every tile base
    uint64_t fixmask;        // live-tile passes: physical bits still equal to the basis bits (0 = all tiles)
    uint64_t zmask, zval;    // live-tile passes: window bits first windowed here; amplitudes off zval are zero (not read)
    double* bins;            // fused marginal: 2^nbq fp64 bins (global)
    int nbq, fflags;         // fflags: 1 = synthesise the first load, 2 = fused marginal
    int8_t bin_pos[16];      // physical bit of output bit k (k = 0 is the MSB)
    uint16_t regbin[TILE_NREG];  // bin bits contributed by the last segment's register index
    // output permutation (TileSpec::operm): the last segment stores window bit b
    // at physical wpos[operm[b]]; tph_out = its thread-nibble offsets
    int has_operm;
    int8_t operm[TILE_W];
    uint64_t tph_out[TILE_TCH][16];
    // checked JIT kernels (QJ_JIT_CHECK=1; compute-sanitizer is not available on
    // this pool): every global access is bounds-checked against namps and a
    // violation sets *chk instead of touching memory (qj_sync reports it)
    uint64_t namps;
    unsigned int* chk;
};

}  // namespace qj
