// util.cu -- unit-test / utility kernels (model classification with ids,
// verify_sorted + multiset_hash, decode) and one-time kernel setup.
#include <algorithm>
#include <cstdlib>

#include "kernels_common.cuh"

namespace lsort_dev {

template <bool IN_F64>
__global__ void __launch_bounds__(256) k_classify_ids(const uint8_t* model, const void* keys, uint64_t n, uint32_t* ids,
                                                     uint16_t* ids16, unsigned long long* hist) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    __shared__ uint32_t sh[kMaxNB];
    uint8_t* msm = (uint8_t*)smem_u4;
    load_model_smem(model, msm);
    Classifier C;
    C.init(msm);
    if (hist) {
        for (uint32_t b = threadIdx.x; b < C.nb; b += 256) sh[b] = 0;
        __syncthreads();
    }
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        uint64_t k = load_key(keys, i, IN_F64);
        const uint32_t c = C.classify_any(k);
        const uint32_t b = c & 0x7fffffffu;
        if (ids) ids[i] = b;
        if (ids16) ids16[i] = (c >> 31) ? kNoMove : (uint16_t)b;
        if (hist) atomicAdd(&sh[b], 1u);
    }
    if (hist) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < C.nb; b += 256)
            if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
    }
}

// Alg. 4 learned_pivots_for_samplesort: per learned cell
// the largest key and whether the cell was hit (per-CTA shared maxima, one
// global atomic per hit cell per CTA). The host drops empty cells.
template <bool IN_F64>
__global__ void __launch_bounds__(256) k_learned_pivots(const uint8_t* model, const void* keys, uint64_t n,
                                                       unsigned long long* gmax, unsigned int* ghit) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    __shared__ unsigned long long smax[kMaxNB];
    __shared__ unsigned int shit[kMaxNB];
    uint8_t* msm = (uint8_t*)smem_u4;
    load_model_smem(model, msm);
    Classifier C;
    C.init(msm);
    for (uint32_t b = threadIdx.x; b < C.nb; b += 256) { smax[b] = 0; shit[b] = 0; }
    __syncthreads();
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        const uint64_t k = load_key(keys, i, IN_F64);
        const uint32_t g = C.classify<kLearned>(k);
        atomicMax(&smax[g], (unsigned long long)k);
        shit[g] = 1u;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < C.nb; b += 256)
        if (shit[b]) {
            atomicMax(&gmax[b], smax[b]);
            atomicOr(&ghit[b], 1u);
        }
}

// P(A <= p) * N for each pivot (upper bound over the sorted keys, compared encoded)
template <bool F64>
__global__ void k_rank_le(const void* sorted, uint64_t n, const uint64_t* pivots, uint32_t np, uint64_t* ranks) {
    griddep_wait();
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const uint64_t p = pivots[i];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (load_key(sorted, mid, F64) <= p) lo = mid + 1;
        else hi = mid;
    }
    ranks[i] = lo;
}

// verify_sorted + multiset_hash (verify.hpp:17-29)
template <bool F64>
__global__ void __launch_bounds__(256) k_verify(const void* keys, uint64_t n, Ctrl* ctrl) {
    griddep_wait();
    __shared__ uint64_t red[8];
    uint64_t first = ~0ull, h = 0;
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        uint64_t k = load_key(keys, i, F64);
        h += splitmix64(k);
        if (i > 0 && load_key(keys, i - 1, F64) > k && i < first) first = i;
    }
    first = block_reduce_min<256>(first, red);
    h = block_reduce_sum_u64<256>(h, red);
    if (threadIdx.x == 0) {
        if (first != ~0ull) atomicMin(&ctrl->verify_first, (unsigned long long)first);
        atomicAdd(&ctrl->verify_hash, (unsigned long long)h);
    }
}

__global__ void k_decode(uint64_t* keys, uint64_t n) {
    griddep_wait();
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
        ((double*)keys)[i] = decode(keys[i]);
}

// Small host<->device transfers as kernels over mapped pinned memory (UVA):
// used while the copy engines stream whole arrays (lsort_cuda_sort_batch), so
// a level's control traffic does not queue behind a multi-MB copy.
__global__ void __launch_bounds__(256) k_copy_bytes(uint8_t* dst, const uint8_t* src, size_t bytes) {
    griddep_wait();
    const size_t tid = blockIdx.x * 256ull + threadIdx.x, step = gridDim.x * 256ull;
    if ((((uintptr_t)dst | (uintptr_t)src | bytes) & 15) == 0) {
        for (size_t i = tid; i < bytes / 16; i += step) ((uint4*)dst)[i] = ((const uint4*)src)[i];
    } else {
        for (size_t i = tid; i < bytes; i += step) dst[i] = src[i];
    }
}

void launch_copy_bytes(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!bytes) return;
    const int grid = (int)std::min<size_t>((bytes + 4095) / 4096, 64);
    pdl(k_copy_bytes, grid, 256, 0, st, (uint8_t*)dst, (const uint8_t*)src, bytes);
}

static int g_num_sms = 148;
bool pdl_enabled() {
    static const bool on = getenv("LSORT_NO_PDL") == nullptr;
    return on;
}
int num_sms() { return g_num_sms; }

void partition_init(int optin);
void models_init(int optin);
void basecase_init(int optin);
void cluster_init(int optin);
void classic_init(int optin);

void kernels_init() {
    static bool done = false;
    if (done) return;
    done = true;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    partition_init(optin);
    models_init(optin);
    basecase_init(optin);
    cluster_init(optin);
    classic_init(optin);
    allow_smem(k_classify_ids<true>, optin);
    allow_smem(k_classify_ids<false>, optin);
    allow_smem(k_learned_pivots<true>, optin);
    allow_smem(k_learned_pivots<false>, optin);
}

void launch_learned_pivots(const uint8_t* model, const void* keys, uint64_t n, int in_f64, unsigned long long* gmax,
                           unsigned int* ghit, int payload, cudaStream_t st) {
    const size_t sm = sizeof(ModelHdr) + (size_t)payload;
    const int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 4);
    if (in_f64) pdl(k_learned_pivots<true>, grid, 256, sm, st, model, keys, n, gmax, ghit);
    else pdl(k_learned_pivots<false>, grid, 256, sm, st, model, keys, n, gmax, ghit);
}

void launch_rank_le(const void* sorted, uint64_t n, int f64, const uint64_t* pivots, uint32_t np, uint64_t* ranks,
                    cudaStream_t st) {
    const int grid = (int)((np + 127) / 128);
    if (f64) pdl(k_rank_le<true>, grid, 128, 0, st, sorted, n, pivots, np, ranks);
    else pdl(k_rank_le<false>, grid, 128, 0, st, sorted, n, pivots, np, ranks);
}

void launch_classify_ids(const uint8_t* model, const void* keys, uint64_t n, int in_f64, uint32_t* ids,
                         uint16_t* ids16, unsigned long long* hist, int payload, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)g_num_sms * 8);
    if (grid < 1) grid = 1;
    size_t sm = sizeof(ModelHdr) + (size_t)payload + 16;
    if (in_f64) pdl(k_classify_ids<true>, grid, 256, sm, st, model, keys, n, ids, ids16, hist);
    else pdl(k_classify_ids<false>, grid, 256, sm, st, model, keys, n, ids, ids16, hist);
}

void launch_verify(const void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)g_num_sms * 8);
    if (grid < 1) grid = 1;
    if (f64) pdl(k_verify<true>, grid, 256, 0, st, keys, n, ctrl);
    else pdl(k_verify<false>, grid, 256, 0, st, keys, n, ctrl);
}

void launch_decode(uint64_t* keys, uint64_t n, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)g_num_sms * 8);
    if (grid < 1) grid = 1;
    pdl(k_decode, grid, 256, 0, st, keys, n);
}

}  // namespace lsort_dev
