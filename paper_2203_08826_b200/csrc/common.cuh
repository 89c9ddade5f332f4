// common.cuh -- device helpers shared by the sm_100a kernels of libqj.
//
// Layout: the state is 2^n_local interleaved
// complex amplitudes; qubit q <-> bit (n-1-q) of the index (reading R1).  Each
// thread moves 16-byte vectors: one complex128 amplitude or two complex64
// amplitudes (bit 0 then lives inside the vector).  A warp covers 32
// consecutive vectors = 512 contiguous bytes, so bits [0, LB) with
// LB = V + 5 are "low" (vector + lane) bits and every bit >= LB is an "outer"
// bit owned by a register index or the loop counter.
#pragma once

#ifdef __CUDACC_RTC__
// NVRTC (run-time compiled tile kernels, tile_jit.cpp): no system headers.
typedef unsigned long long uint64_t;
typedef unsigned int uint32_t;
typedef unsigned short uint16_t;
typedef unsigned char uint8_t;
typedef long long int64_t;
typedef short int16_t;
typedef signed char int8_t;
typedef int int32_t;
#else
#include <cuda_runtime.h>
#include <stdint.h>
#endif

namespace qj {

template <typename R>
struct Cx {
    R re, im;
};

template <typename R>
__host__ __device__ __forceinline__ Cx<R> cmul(Cx<R> a, Cx<R> b) {
    return Cx<R>{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}

// acc += a * b  (4 FMAs)
template <typename R>
__device__ __forceinline__ void cfma(Cx<R>& acc, Cx<R> a, Cx<R> b) {
    acc.re = fma(a.re, b.re, acc.re);
    acc.re = fma(-a.im, b.im, acc.re);
    acc.im = fma(a.re, b.im, acc.im);
    acc.im = fma(a.im, b.re, acc.im);
}

template <typename R>
struct VecT;
template <>
struct VecT<double> {
    using type = double2;  // one complex128 amplitude
    static constexpr int V = 0;
};
template <>
struct VecT<float> {
    using type = float4;  // two complex64 amplitudes (bit 0 inside the vector)
    static constexpr int V = 1;
};

__device__ __forceinline__ void unpack(const double2& v, Cx<double> (&a)[1]) { a[0] = {v.x, v.y}; }
__device__ __forceinline__ void unpack(const float4& v, Cx<float> (&a)[2]) {
    a[0] = {v.x, v.y};
    a[1] = {v.z, v.w};
}
__device__ __forceinline__ double2 pack(const Cx<double> (&a)[1]) { return make_double2(a[0].re, a[0].im); }
__device__ __forceinline__ float4 pack(const Cx<float> (&a)[2]) {
    return make_float4(a[0].re, a[0].im, a[1].re, a[1].im);
}

// 128-bit global accesses.  The state is read and written exactly once per
// pass by exactly one thread, so the streaming (evict-first) hints apply for
// states larger than L2; for L2-resident states they are harmless.
__device__ __forceinline__ double2 ldv(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ldv(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void stv(double2* p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void stv(float4* p, float4 v) { __stcs(p, v); }

// Store one amplitude at amplitude index idx (used when a vector cannot be
// assembled: complex64 passes that write amplitudes one by one).
__device__ __forceinline__ void store_amp(void* psi, uint64_t idx, Cx<double> o) {
    __stcs(reinterpret_cast<double2*>(psi) + idx, make_double2(o.re, o.im));
}
__device__ __forceinline__ void store_amp(void* psi, uint64_t idx, Cx<float> o) {
    __stcs(reinterpret_cast<float2*>(psi) + idx, make_float2(o.re, o.im));
}

__device__ __forceinline__ Cx<double> load_amp(const Cx<double>* psi, uint64_t idx) {
    const double2 v = __ldcs(reinterpret_cast<const double2*>(psi) + idx);
    return Cx<double>{v.x, v.y};
}
__device__ __forceinline__ Cx<float> load_amp(const Cx<float>* psi, uint64_t idx) {
    const float2 v = __ldcs(reinterpret_cast<const float2*>(psi) + idx);
    return Cx<float>{v.x, v.y};
}

template <typename R>
__device__ __forceinline__ Cx<R> shfl_xor(Cx<R> v, int m) {
    return Cx<R>{__shfl_xor_sync(0xffffffffu, v.re, m), __shfl_xor_sync(0xffffffffu, v.im, m)};
}

// Bit insertion: open a 0 at bit position p.
__host__ __device__ __forceinline__ uint64_t insert_zero(uint64_t x, int p) {
    const uint64_t lo = x & ((1ull << p) - 1ull);
    return ((x >> p) << (p + 1)) | lo;
}

constexpr int MAXB = 48;  // max inserted positions per pass

}  // namespace qj
