// Microbenchmark: shared-memory histogram strategies on B200.
//   mode 0: plain atomicAdd per key
//   mode 1: __match_any_sync warp aggregation + leader atomicAdd
//   mode 2: atomicAdd with return (rank), plain
//   mode 3: match_any rank (leader add + shfl)
//   mode 4: no histogram (load + bucket compute only)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t bucket_of(uint64_t k, uint32_t mask) {
    return (uint32_t)((k * 0x9e3779b97f4a7c15ull) >> 40) & mask;
}

template <int MODE>
__global__ void __launch_bounds__(256) k(const uint64_t* keys, uint64_t n, uint32_t mask, unsigned* out) {
    __shared__ uint32_t h[2048];
    for (int i = threadIdx.x; i < 2048; i += 256) h[i] = 0;
    __syncthreads();
    uint32_t acc = 0;
    const int lane = threadIdx.x & 31;
    for (uint64_t base = (uint64_t)blockIdx.x * 4096; base < n; base += (uint64_t)gridDim.x * 4096) {
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
            uint64_t i = base + threadIdx.x + j * 256;
            uint64_t key = i < n ? keys[i] : 0;
            uint32_t b = bucket_of(key, mask);
            if (MODE == 0) atomicAdd(&h[b], 1u);
            else if (MODE == 1) {
                unsigned peers = __match_any_sync(0xffffffffu, b);
                if (lane == __ffs(peers) - 1) atomicAdd(&h[b], (unsigned)__popc(peers));
            } else if (MODE == 2) {
                acc += atomicAdd(&h[b], 1u);
            } else if (MODE == 3) {
                unsigned peers = __match_any_sync(0xffffffffu, b);
                int leader = __ffs(peers) - 1;
                uint32_t old = 0;
                if (lane == leader) old = atomicAdd(&h[b], (unsigned)__popc(peers));
                old = __shfl_sync(0xffffffffu, old, leader);
                acc += old + __popc(peers & ((1u << lane) - 1));
            } else {
                acc += b;
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(out, h[0] + acc);
}

int main() {
    const uint64_t n = 100000000;
    uint64_t* d;
    unsigned* o;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 4);
    // keys: i (uniform buckets after hashing); second run: all equal
    uint64_t* h = new uint64_t[n];
    for (uint64_t i = 0; i < n; ++i) h[i] = i;
    cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int dist = 0; dist < 2; ++dist) {
        if (dist == 1) cudaMemset(d, 0, n * 8);
        for (uint32_t mask : {1023u, 255u, 0u}) {
            for (int mode = 0; mode < 5; ++mode) {
                float best = 1e9;
                for (int r = 0; r < 4; ++r) {
                    cudaEventRecord(a);
                    switch (mode) {
                    case 0: k<0><<<nsm * 8, 256>>>(d, n, mask, o); break;
                    case 1: k<1><<<nsm * 8, 256>>>(d, n, mask, o); break;
                    case 2: k<2><<<nsm * 8, 256>>>(d, n, mask, o); break;
                    case 3: k<3><<<nsm * 8, 256>>>(d, n, mask, o); break;
                    default: k<4><<<nsm * 8, 256>>>(d, n, mask, o); break;
                    }
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    best = ms < best ? ms : best;
                }
                printf("keys=%s buckets=%4u mode=%d  %.3f ms  (%.1f GB/s read)\n", dist ? "equal" : "spread", mask + 1,
                       mode, best, n * 8 / best / 1e6);
            }
        }
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
