// membench2.cu -- pipeline ceiling of a one-CTA-per-SM window tile pass (not
// part of the library).  Tile = 2^W 16-byte amplitudes whose index bits are the
// low L bits plus W-L bits from bit P; 2^(W-4) threads x 16 registers.
//   mode 0: registers <- HBM directly, compute, registers -> HBM
//   mode 1: the next tile is prefetched with cp.async into a 2^W-amplitude SMEM
//           buffer as soon as the current one has been read out of it; the
//           SMEM transposes run through a separate half-size buffer in two
//           rounds (one stable thread bit selects the round).
// ntr dummy transposes and nfma dependent-free DFMA pairs per amplitude
// emulate the gate work.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench2 tools/membench2.cu
//   ./membench2 n W L P mode ntr nfma
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int b) {
    const uint64_t lo = x & ((1ull << b) - 1);
    return ((x >> b) << (b + 1)) | lo;
}
__device__ __forceinline__ void cp16(void* s, const void* g) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g));
}

struct Args {
    double2* psi;
    uint64_t ntiles;
    int W, L, P, mode, ntr, nfma;
    double one, zero;
};

template <int T>  // threads
__global__ void __launch_bounds__(T, 1) tile_pipe(Args a) {
    extern __shared__ __align__(16) double2 sm[];
    const int tid = threadIdx.x;
    const int H = a.W - a.L;
    double2* pre = sm;                    // 2^W prefetch buffer
    double2* tr = a.mode == 1 ? sm + (1 << a.W) : sm;  // 2^(W-1) transpose buffer
    auto base = [&](uint64_t tile) {
        uint64_t tb = tile;
        for (int i = 0; i < a.L; ++i) tb = insert_zero(tb, i);
        for (int i = 0; i < H; ++i) tb = insert_zero(tb, a.P + i);
        return tb;
    };
    auto addr = [&](uint64_t tb, int r) {
        const uint32_t w = (uint32_t)tid | ((uint32_t)r << (a.W - 4));
        const uint64_t lo = w & ((1u << a.L) - 1), hi = w >> a.L;
        return tb | lo | (hi << a.P);
    };
    auto prefetch = [&](uint64_t tile) {
        const uint64_t tb = base(tile);
#pragma unroll
        for (int r = 0; r < 16; ++r) cp16(pre + (tid | (r << (a.W - 4))), a.psi + addr(tb, r));
        asm volatile("cp.async.commit_group;\n" ::);
    };
    uint64_t tile = blockIdx.x;
    if (a.mode == 1 && tile < a.ntiles) prefetch(tile);
    for (; tile < a.ntiles; tile += gridDim.x) {
        double2 v[16];
        const uint64_t tb = base(tile);
        if (a.mode == 1) {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
            __syncthreads();
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = pre[tid | (r << (a.W - 4))];
            __syncthreads();
            if (tile + gridDim.x < a.ntiles) prefetch(tile + gridDim.x);
        } else {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = __ldcg(a.psi + addr(tb, r));
        }
        for (int t = 0; t < a.ntr; ++t) {
            // two rounds: threads with bit (W-5) == round write and read back
            for (int round = 0; round < 2; ++round) {
                const bool mine = ((tid >> (a.W - 5)) & 1) == round;
                const int lt = tid & ((1 << (a.W - 5)) - 1);
                if (mine)
#pragma unroll
                    for (int r = 0; r < 16; ++r) tr[(lt * 16 + r) ^ ((lt >> 3) & 15)] = v[r];
                __syncthreads();
                if (mine)
#pragma unroll
                    for (int r = 0; r < 16; ++r) v[r] = tr[(((r + t) & 15) * (1 << (a.W - 5)) + lt) ^ 0];
                __syncthreads();
            }
        }
        for (int f = 0; f < a.nfma; ++f)
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                v[r].x = fma(v[r].x, a.one, a.zero);
                v[r].y = fma(v[r].y, a.one, a.zero);
            }
#pragma unroll
        for (int r = 0; r < 16; ++r) __stcg(a.psi + addr(tb, r), v[r]);
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 30;
    Args a{};
    a.W = argc > 2 ? atoi(argv[2]) : 13;
    a.L = argc > 3 ? atoi(argv[3]) : 4;
    a.P = argc > 4 ? atoi(argv[4]) : 21;
    a.mode = argc > 5 ? atoi(argv[5]) : 1;
    a.ntr = argc > 6 ? atoi(argv[6]) : 0;
    a.nfma = argc > 7 ? atoi(argv[7]) : 0;
    const int reps = 5;
    const size_t bytes = (size_t)16 << n;
    double2* psi;
    if (cudaMalloc(&psi, bytes) != cudaSuccess) return 1;
    cudaMemset(psi, 0, bytes);
    a.psi = psi;
    a.one = 1.0;
    a.zero = 0.0;
    a.ntiles = 1ull << (n - a.W);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = a.mode == 1 ? (size_t)16 * ((1 << a.W) + (1 << (a.W - 1))) : (size_t)16 * (1 << (a.W - 1));
    auto launch = [&]() {
        if (a.W == 13) {
            cudaFuncSetAttribute(tile_pipe<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            tile_pipe<512><<<sms, 512, smem>>>(a);
        } else {
            cudaFuncSetAttribute(tile_pipe<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            tile_pipe<256><<<sms, 256, smem>>>(a);
        }
    };
    launch();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float sum = 0;
    for (int i = 0; i < reps; ++i) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        sum += ms;
    }
    const cudaError_t err = cudaGetLastError();
    printf("{\"W\": %d, \"L\": %d, \"P\": %d, \"mode\": %d, \"ntr\": %d, \"nfma\": %d, \"ms\": %.3f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           a.W, a.L, a.P, a.mode, a.ntr, a.nfma, sum / reps, 2.0 * bytes / (sum / reps * 1e-3) / 1e9,
           cudaGetErrorString(err));
    return 0;
}
