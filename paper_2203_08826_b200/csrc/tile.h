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

#include <string>
#include <vector>

#include "qj_internal.h"
#include "tile_abi.h"

namespace qj {

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
    uint64_t gbase = 0;  // sharded states: (shard index) << n_local, OR-ed into predicate indices
    // qj_simulate (JIT kernels only): the first pass can synthesise |basis>
    // instead of loading, the last pass can accumulate the marginal of the
    // listed physical bits (first = MSB of the bin index) into `bins`.
    bool synth = false;
    uint64_t synth_index = 0;
    // qj_simulate, later passes of a |basis> run: bits no earlier pass has
    // targeted still equal the basis bits (zero elsewhere), so only the tiles
    // whose fixed bits match are live; ntiles counts those, bit-inserted
    uint64_t fix_mask = 0, fix_val = 0;
    // ... and of each live tile only the amplitudes whose newly windowed bits
    // (zero_mask) equal the basis bits are nonzero: the rest load as zeros
    uint64_t zero_mask = 0, zero_val = 0;
    int nbins_q = 0;            // 0 = no fused marginal
    int8_t bin_pos[16] = {};
    double* bins = nullptr;
    int w = 0;
    int wpos[TILE_W] = {};
    // store in the last segment's own layout (no store transpose): window bit b
    // is written to window position operm[b]; the planner relabels the qubit
    // map accordingly (like an uncontrolled SWAP, R21).  identity when !operm_on
    bool operm_on = false;
    int8_t operm[TILE_W] = {};
    std::vector<TSeg> segs;
    std::vector<HOp> ops;        // ops in order; segs[].op0/op1 index into it
};

// Pinned-host + device ring for the per-pass program buffers.
struct TileStaging {
    static constexpr int kSlots = 8;
    static constexpr size_t kBytes = 512 * 1024;
    unsigned char* host = nullptr;  // pinned, kSlots * kBytes
    unsigned char* dev = nullptr;   // device, kSlots * kBytes
    cudaEvent_t ev[kSlots] = {};
    int next = 0;
    cudaError_t init();
    void release();
};

template <typename R>
cudaError_t run_tile(const TileSpec& t, void* psi, int nl, cudaStream_t st, TileStaging& stg, LaunchStats& ls);

// A tile pass lowered once with a persistent device program buffer, for
// cached circuits replayed (and captured into CUDA graphs) without re-lowering
// or host->device copies.
struct PreparedTile {
    std::vector<unsigned char> args;  // TileArgs<R> bytes (tables -> dev)
    void* dev = nullptr;              // device program buffer (owned)
    void* jit = nullptr;              // JIT function or nullptr (interpreter)
    size_t smem = 0;
    unsigned grid = 0;
    int threads = TILE_THREADS;  // block size (JIT ring form: 2 x TILE_THREADS)
    int amp_bytes = 16;
};
template <typename R>
cudaError_t tile_prepare(const TileSpec& t, void* psi, int nl, PreparedTile& out);
cudaError_t tile_launch_prepared(const PreparedTile& p, cudaStream_t st, LaunchStats& ls);
void tile_release(PreparedTile& p);

// Host lowering of a planned pass into kernel parameters + program buffer
// (false when it exceeds a capacity).
template <typename R>
bool lower_tile(const TileSpec& t, int nl, TileArgs<R>* a, std::vector<unsigned char>& blob);

// Tooling (qj_debug_tile_sources): write the JIT source of a lowered pass to
// `path` and, with `compile`, compile it with NVRTC for sm_100a (no GPU
// needed); returns false with *err set on a lowering or compile failure.
template <typename R>
bool tile_jit_debug_source(const TileSpec& t, int nl, const char* path, bool compile, std::string* err);

// Whether a planned pass lowers within the kernel's capacities.
bool tile_fits(const TileSpec& t, int nl, int amp_bytes);

}  // namespace qj
