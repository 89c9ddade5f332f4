// dense_tc.h -- complex64 dense 5-qubit passes on the tensor cores
// (tcgen05.mma kind::tf32, 3xTF32; dense_tc.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "qj_internal.h"

namespace qj {

struct TcArgs {
    float2 u[32][32];     // U, row-major, first-listed target = MSB of the row / column index (R3)
    uint64_t moff[32];    // member j -> offset of its target bits
    int nins;             // sorted target + fixed positions (bit insertion)
    int ins_pos[16];
    uint64_t fix_val;     // fixed bits (controls = 1)
    uint64_t ngroups;     // 2^(nl - nins)
    void* psi;
    // staged form (a target or fixed bit below bit 5: a thread's own members
    // would be uncoalesced): a tile's 4096 amplitudes, indexed by L whose 12
    // bits are the 7 lowest free positions and the 5 target positions in
    // ascending physical order, move through shared memory cooperatively
    int staged;
    int lpos_row[7];      // physical position of L bits 0..6 (a thread's row index)
    uint32_t w_row[7];    // staging index weight of L bits 0..6
    uint64_t addr_m[32];  // physical offset of L bits 7..11 (m = L >> 7)
    uint32_t sidx_m[32];  // staging index of L bits 7..11
};

// QJ_TC=0 keeps every dense pass on the CUDA cores.
bool dense_tc_enabled();
// A dense pass the tensor-core kernel takes: 5 targets, every member touched,
// at least one 128-group tile.
bool dense_tc_supports(const Pass& p, int nl);
cudaError_t run_dense_tc(const Pass& p, void* psi, int nl, cudaStream_t st, LaunchStats& ls);

}  // namespace qj
