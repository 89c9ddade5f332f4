// dist.cu -- NCCL loader and the exchange pack / unpack / copy kernels (dist.h).
#include <dlfcn.h>

#include <mutex>

#include "common.cuh"
#include "dist.h"

namespace qj {

const NcclApi* nccl_api(const char** why) {
    static NcclApi api;
    static std::once_flag once;
    static const char* err = nullptr;
    std::call_once(once, [] {
        // prefer the copy torch already loaded (its communicators live there)
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = "libnccl.so.2 not found";
            return;
        }
#define QJ_SYM(field, name)                                              \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
    if (!api.field) {                                                    \
        err = "NCCL symbol " name " missing";                            \
        return;                                                          \
    }
        QJ_SYM(Send, "ncclSend");
        QJ_SYM(Recv, "ncclRecv");
        QJ_SYM(GroupStart, "ncclGroupStart");
        QJ_SYM(GroupEnd, "ncclGroupEnd");
        QJ_SYM(AllReduce, "ncclAllReduce");
        QJ_SYM(CommUserRank, "ncclCommUserRank");
        QJ_SYM(CommCount, "ncclCommCount");
        QJ_SYM(GetErrorString, "ncclGetErrorString");
#undef QJ_SYM
        api.ok = true;
    });
    if (!api.ok) {
        if (why) *why = err;
        return nullptr;
    }
    return &api;
}

// Half-index h (0 .. 2^(nl-1)) <-> amplitude index with local bit L = half_bit.
template <typename T>
__global__ void half_pack_kernel(const T* __restrict__ state, T* __restrict__ buf, int L, int hb, uint64_t h0,
                                 uint64_t count) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = insert_zero(h0 + i, L) | ((uint64_t)hb << L);
        buf[i] = state[idx];
    }
}
template <typename T>
__global__ void half_unpack_kernel(T* __restrict__ state, const T* __restrict__ buf, int L, int hb, uint64_t h0,
                                   uint64_t count) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t idx = insert_zero(h0 + i, L) | ((uint64_t)hb << L);
        state[idx] = buf[i];
    }
}
__global__ void copy16_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, uint64_t n16) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (uint64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

static unsigned grid_of(uint64_t n) {
    uint64_t b = (n + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148ull * 16 ? 148ull * 16 : b));
}

cudaError_t launch_half_pack(const void* state, void* buf, int amp_bytes, int L, int hb, uint64_t h0, uint64_t count,
                             cudaStream_t st) {
    if (amp_bytes == 16)
        half_pack_kernel<double2><<<grid_of(count), 256, 0, st>>>(static_cast<const double2*>(state),
                                                                  static_cast<double2*>(buf), L, hb, h0, count);
    else
        half_pack_kernel<float2><<<grid_of(count), 256, 0, st>>>(static_cast<const float2*>(state),
                                                                 static_cast<float2*>(buf), L, hb, h0, count);
    return cudaGetLastError();
}

cudaError_t launch_half_unpack(void* state, const void* buf, int amp_bytes, int L, int hb, uint64_t h0,
                               uint64_t count, cudaStream_t st) {
    if (amp_bytes == 16)
        half_unpack_kernel<double2><<<grid_of(count), 256, 0, st>>>(static_cast<double2*>(state),
                                                                    static_cast<const double2*>(buf), L, hb, h0, count);
    else
        half_unpack_kernel<float2><<<grid_of(count), 256, 0, st>>>(static_cast<float2*>(state),
                                                                   static_cast<const float2*>(buf), L, hb, h0, count);
    return cudaGetLastError();
}

cudaError_t launch_copy(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    const uint64_t n16 = bytes / 16;
    if (n16) copy16_kernel<<<grid_of(n16), 256, 0, st>>>(static_cast<uint4*>(dst), static_cast<const uint4*>(src), n16);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess && bytes % 16)  // tail (e.g. one complex64 amplitude of a 2-amplitude shard)
        e = cudaMemcpyAsync(static_cast<char*>(dst) + n16 * 16, static_cast<const char*>(src) + n16 * 16, bytes % 16,
                            cudaMemcpyDeviceToDevice, st);
    return e;
}

}  // namespace qj
