// Write-out microbenchmark: staged 4 Ki-key tiles (256 runs of 16 keys) stored
// to per-bucket cursors either by warp stores (sbid + delta lookups, as in
// k_scatter) or by one TMA bulk store (cp.async.bulk) per run.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2307_08637_b200/csrc tma_store_bench.cu -o /tmp/tsb
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tma.cuh"
using namespace lsort_dev;

constexpr int NT = 512, TILE = 4096, NB = 256, RUN = TILE / NB, TPS = 244;  // tiles per segment

__device__ __forceinline__ uint64_t dst_of(uint64_t t, uint32_t b, uint32_t shift) {
    const uint64_t s = t / TPS, k = t % TPS;
    return s * (uint64_t)TPS * TILE + (uint64_t)b * (TPS * RUN) + k * RUN + shift;
}

template <int MODE>
__global__ void __launch_bounds__(NT, 2) k_write(uint64_t* dst, uint64_t ntiles, uint32_t shift) {
    extern __shared__ uint4 smem_u4[];
    uint64_t (*stage)[TILE + 2 * NB] = (uint64_t (*)[TILE + 2 * NB])smem_u4;
    long long* delta = (long long*)(stage[2]);
    uint16_t* sbid = (uint16_t*)(delta + NB);
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x, t0 = blockIdx.x * per, t1 = min(t0 + per, ntiles);
    for (uint64_t t = t0; t < t1; ++t) {
        const int tb = (int)((t - t0) & 1);
        uint64_t* sk = stage[tb];
        if (MODE >= 1 && threadIdx.x < NB) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncthreads();
        // staging: random-ish positions (a permutation of the tile)
#pragma unroll
        for (int q = 0; q < TILE / NT; ++q) {
            const uint32_t j = threadIdx.x + q * NT;
            uint32_t pos = (j * 2654435761u) & (TILE - 1);
            if (MODE == 2) pos = (pos / RUN) * (RUN + 2) + (uint32_t)(dst_of(t, pos / RUN, shift) & 1) + pos % RUN;
            sk[pos] = t * TILE + j;
            if (MODE == 0) sbid[pos] = (uint16_t)(pos / RUN);
        }
        if (threadIdx.x < NB) delta[threadIdx.x] = (long long)dst_of(t, threadIdx.x, shift) - threadIdx.x * RUN;
        if (MODE >= 1) fence_proxy_async_smem();
        __syncthreads();
        if (MODE == 0) {
#pragma unroll
            for (int q = 0; q < TILE / NT; ++q) {
                const uint32_t j = threadIdx.x + q * NT;
                dst[(long long)j + delta[sbid[j]]] = sk[j];
            }
        } else if (MODE == 2 && threadIdx.x < NB) {
            const uint32_t b = threadIdx.x;
            const uint64_t d = dst_of(t, b, shift);
            const uint32_t h = (uint32_t)(d & 1), n = RUN;
            const uint64_t* src = sk + b * (RUN + 2) + h;  // staged at the destination's parity
            if (h) dst[d] = src[0];
            const uint32_t body = (n - h) & ~1u;
            if (body) tma_store_1d(dst + d + h, src + h, body * 8);
            if (h + body < n) dst[d + n - 1] = src[n - 1];
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        } else if (MODE == 1 && threadIdx.x < NB) {
            const uint32_t b = threadIdx.x;
            const uint64_t d = dst_of(t, b, shift);
            uint32_t h = (uint32_t)(d & 1), n = RUN;  // 16-byte aligned body
            if (h) dst[d] = sk[b * RUN];
            const uint32_t body = (n - h) & ~1u;
            if (body) tma_store_1d(dst + d + h, sk + b * RUN + h, body * 8);
            if (h + body < n) dst[d + n - 1] = sk[b * RUN + n - 1];
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (MODE >= 1 && threadIdx.x < NB) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const uint64_t ntiles = 122000, n = ntiles * TILE + 64;
    uint64_t* dst;
    cudaMalloc(&dst, n * 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const size_t sm = 2 * (TILE + 2 * NB) * 8 + NB * 8 + TILE * 2;
    cudaFuncSetAttribute(k_write<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_write<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(k_write<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    for (int mode = 0; mode < 3; ++mode)
        for (uint32_t shift = 0; shift < 2; ++shift) {
            for (int r = 0; r < 4; ++r) {
                cudaEventRecord(a);
                if (mode == 0) k_write<0><<<296, NT, sm>>>(dst, ntiles, shift);
                else if (mode == 1) { if (shift) continue; k_write<1><<<296, NT, sm>>>(dst, ntiles, shift); }
                else k_write<2><<<296, NT, sm>>>(dst, ntiles, shift);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r == 3)
                    printf("mode %s shift %u: %.3f ms  %.1f GB/s written (%s)\n", mode == 2 ? "tma-parity" : (mode ? "tma" : "stg"), shift, ms,
                           ntiles * TILE * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
            }
        }
    return 0;
}
