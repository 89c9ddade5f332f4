// dist.h -- multi-GPU layer of libqj: one process per GPU, the
// state sharded on its top g = log2(P) "global" qubits, and local<->global
// qubit swaps executed as pairwise exchanges over NCCL (NVLink 5 / NVSwitch).
//
// NCCL is the one torch already loaded (the communicator comes from
// ProcessGroupNCCL::_comm_ptr()); it is resolved with dlopen/dlsym at first
// use, so libqj loads (and its CPU tests run) without NCCL present.
//
// Exchange of global bit j with local bit L (the paper's multi-device scheme,
// PAPER.md:469-489, redesigned): rank r and partner r ^ (1 << j) trade the
// halves of their shards whose local bit L differs from their own global bit
// j: rank r with global bit v = (r >> j) & 1 sends (and receives into) the
// amplitudes whose local bit L equals 1 - v.  Halves move in chunks through a
// two-slot staging ring (send and receive buffers must not alias); when L is
// the top local bit the half is contiguous and is sent in place, otherwise it
// is packed / unpacked by kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <nccl.h>

namespace qj {

struct NcclApi {
    bool ok = false;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// Loads NCCL on first call; returns nullptr (and a message) if unavailable.
const NcclApi* nccl_api(const char** why);

// The exchange rule (exported as qj_exchange_peer for the CPU tests).
struct ExchangeSpec {
    int peer;       // partner rank
    int half_bit;   // value of local bit L of the amplitudes this rank sends / receives
};
inline ExchangeSpec exchange_spec(int rank, int gbit) {
    ExchangeSpec e;
    e.peer = rank ^ (1 << gbit);
    e.half_bit = 1 - ((rank >> gbit) & 1);
    return e;
}

// Pack / unpack / copy kernels for the exchange (dist.cu).
cudaError_t launch_half_pack(const void* state, void* buf, int amp_bytes, int L, int half_bit, uint64_t h0,
                             uint64_t count, cudaStream_t st);
cudaError_t launch_half_unpack(void* state, const void* buf, int amp_bytes, int L, int half_bit, uint64_t h0,
                               uint64_t count, cudaStream_t st);
cudaError_t launch_copy(void* dst, const void* src, size_t bytes, cudaStream_t st);

}  // namespace qj
