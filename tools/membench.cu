// membench.cu -- memory-path ceiling of the window tile pass (not part of the
// library): an in-place read -> registers -> write of a 2^n x 16-byte buffer in
// 64 KiB tiles whose 12 index bits are the low L bits plus 12-L bits starting
// at bit P (the tile pass's window shape), every other bit enumerating tiles.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench tools/membench.cu
//   ./membench n L P blocks_per_sm order(c|b) [reps]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t insert_zero(uint64_t x, int b) {
    const uint64_t lo = x & ((1ull << b) - 1);
    return ((x >> b) << (b + 1)) | lo;
}

struct Args {
    double2* psi;
    uint64_t ntiles;
    int L, P, blocked, group;
};

// 256 threads x 16 amplitudes; thread bits = tile index bits 0..7, register bits 8..11
template <int MINB>
__global__ void __launch_bounds__(256, MINB) tile_copy(Args a) {
    const int tid = threadIdx.x;
    uint64_t t_lo, t_hi, t_step;
    if (a.blocked) {
        const uint64_t per = (a.ntiles + gridDim.x - 1) / gridDim.x;
        t_lo = blockIdx.x * per;
        t_hi = min(a.ntiles, t_lo + per);
        t_step = 1;
    } else {
        t_lo = blockIdx.x;
        t_hi = a.ntiles;
        t_step = gridDim.x;
    }
    const int H = 12 - a.L;
    for (uint64_t tile = t_lo; tile < t_hi; tile += t_step) {
        // tile base: insert zeros at the window bits (low L and [P, P+H))
        uint64_t tb = tile;
        for (int i = 0; i < a.L; ++i) tb = insert_zero(tb, i);
        for (int i = 0; i < H; ++i) tb = insert_zero(tb, a.P + i);
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t w = (uint32_t)tid | ((uint32_t)r << 8);  // window-local index
            const uint64_t lo = w & ((1u << a.L) - 1), hi = w >> a.L;
            const uint64_t x = tb | lo | (hi << a.P);
            v[r] = __ldcg(a.psi + x);
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t w = (uint32_t)tid | ((uint32_t)r << 8);
            const uint64_t lo = w & ((1u << a.L) - 1), hi = w >> a.L;
            const uint64_t x = tb | lo | (hi << a.P);
            double2 y = v[r];
            asm volatile("" : "+d"(y.x), "+d"(y.y));
            __stcg(a.psi + x, y);
        }
    }
}

// Cluster pairs: the two CTAs of a cluster take sibling tiles (differing in the
// lowest tile bit, i.e. adjacent 128-byte chunks) and meet at a cluster barrier
// before each tile's loads, so DRAM sees both halves of every 256-byte run together.
template <int MINB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, MINB) tile_copy_pair(Args a) {
    const int tid = threadIdx.x;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const uint64_t pairs = a.ntiles / 2, npair_grid = gridDim.x / 2, pid = blockIdx.x / 2;
    const int H = 12 - a.L;
    for (uint64_t pr = pid; pr < pairs; pr += npair_grid) {
        const uint64_t tile = 2 * pr + rank;
        uint64_t tb = tile;
        for (int i = 0; i < a.L; ++i) tb = insert_zero(tb, i);
        for (int i = 0; i < H; ++i) tb = insert_zero(tb, a.P + i);
        if (a.group) {
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
        }
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t w = (uint32_t)tid | ((uint32_t)r << 8);
            const uint64_t lo = w & ((1u << a.L) - 1), hi = w >> a.L;
            v[r] = __ldcg(a.psi + (tb | lo | (hi << a.P)));
        }
#pragma unroll
        for (int r = 0; r < 16; ++r) {
            const uint32_t w = (uint32_t)tid | ((uint32_t)r << 8);
            const uint64_t lo = w & ((1u << a.L) - 1), hi = w >> a.L;
            double2 y = v[r];
            asm volatile("" : "+d"(y.x), "+d"(y.y));
            __stcg(a.psi + (tb | lo | (hi << a.P)), y);
        }
    }
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 30;
    const int L = argc > 2 ? atoi(argv[2]) : 3;
    const int P = argc > 3 ? atoi(argv[3]) : 21;
    const int B = argc > 4 ? atoi(argv[4]) : 2;
    const int blocked = argc > 5 && argv[5][0] == 'b';
    const int reps = argc > 6 ? atoi(argv[6]) : 5;
    const size_t bytes = (size_t)16 << n;
    double2* psi;
    if (cudaMalloc(&psi, bytes) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(psi, 0, bytes);
    Args a{psi, 1ull << (n - 12), L, P, blocked, 0};
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned grid = sms * B;
    const int pairmode = argc > 7 ? atoi(argv[7]) : 0;  // 1: cluster pairs, 2: cluster pairs + barrier
    a.group = pairmode == 2;
    auto launch = [&]() {
        if (pairmode) {
            if (B == 1) tile_copy_pair<1><<<grid, 256>>>(a);
            else tile_copy_pair<2><<<grid, 256>>>(a);
            return;
        }
        switch (B) {
            case 1: tile_copy<1><<<grid, 256>>>(a); break;
            case 2: tile_copy<2><<<grid, 256>>>(a); break;
            case 3: tile_copy<3><<<grid, 256>>>(a); break;
            default: tile_copy<4><<<grid, 256>>>(a); break;
        }
    };
    launch();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f, sum = 0;
    for (int i = 0; i < reps; ++i) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
        sum += ms;
    }
    const cudaError_t err = cudaGetLastError();
    const double gbs = 2.0 * bytes / (sum / reps * 1e-3) / 1e9;
    printf("{\"pair\": %d, \"n\": %d, \"L\": %d, \"P\": %d, \"blocks\": %d, \"order\": \"%s\", \"ms\": %.3f, \"best_ms\": %.3f, \"GBps\": %.1f, \"err\": \"%s\"}\n",
           pairmode, n, L, P, B, blocked ? "b" : "c", sum / reps, best, gbs, cudaGetErrorString(err));
    return 0;
}
