// basecase.cu -- small-segment sorts and equality fills.
//
//   k_base_warp   one warp per segment of <= 512 keys (keys in registers,
//                 range-adaptive MSD counting pass into shared memory,
//                 insertion / warp rank sort of small digits), decode on store.
//   k_base        one CTA per segment of <= 16384 keys (BlockSort).
//   k_small_sort  whole inputs of <= 16384 keys, in place, NaN check first.
//   k_fill        equality buckets / homogeneous segments: value stores only.
// Together they replace radix_base_case_sort + insertion sort
// and mark_homogeneous.
#include <algorithm>

#include "kernels_common.cuh"

namespace lsort_dev {

// ---------------------------------------------------------- warp base case
constexpr int kWNT = 256;
constexpr int kWWarps = kWNT / 32;
constexpr int kWItems = kWarpBaseCap / 32;  // 16 keys per lane
constexpr int kWStack = 32;

struct WarpSmem {
    uint64_t buf[kWarpBaseCap];
    uint32_t hist[257];
    uint32_t n_stk;
    uint32_t stk_off[kWStack];
    uint32_t stk_len[kWStack];
};

__device__ __forceinline__ uint64_t warp_min(uint64_t v) {
    for (int o = 16; o > 0; o >>= 1) { uint64_t w = __shfl_xor_sync(FULL_MASK, v, o); v = w < v ? w : v; }
    return v;
}
__device__ __forceinline__ uint64_t warp_max(uint64_t v) {
    for (int o = 16; o > 0; o >>= 1) { uint64_t w = __shfl_xor_sync(FULL_MASK, v, o); v = w > v ? w : v; }
    return v;
}

__device__ __forceinline__ void insertion_sort(uint64_t* a, uint32_t len) {
    for (uint32_t i = 1; i < len; ++i) {
        uint64_t v = a[i];
        uint32_t j = i;
        while (j > 0 && a[j - 1] > v) { a[j] = a[j - 1]; --j; }
        a[j] = v;
    }
}

// warp rank sort of a[0,len), len <= 256 (8 keys per lane)
__device__ void warp_rank_sort(uint64_t* a, uint32_t len) {
    const int lane = threadIdx.x & 31;
    uint64_t v[8];
    uint32_t r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        uint32_t idx = lane + 32 * q;
        v[q] = idx < len ? a[idx] : ~0ull;
        r[q] = 0;
    }
    for (uint32_t j = 0; j < len; ++j) {
        uint64_t w = a[j];
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] += (w < v[q]) || (w == v[q] && j < (uint32_t)(lane + 32 * q));
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if ((uint32_t)(lane + 32 * q) < len) a[r[q]] = v[q];
    __syncwarp();
}

// One warp-level distribution pass: keys k[] (idx = lane + 32 i < len) into
// W.buf[off, off+len) grouped by (k - min) >> shift; small digits sorted.
__device__ void warp_pass(uint64_t (&k)[kWItems], uint32_t off, uint32_t len, WarpSmem& W) {
    const int lane = threadIdx.x & 31;
    uint64_t mn = ~0ull, mx = 0;
#pragma unroll
    for (int i = 0; i < kWItems; ++i)
        if ((uint32_t)(lane + 32 * i) < len) { mn = k[i] < mn ? k[i] : mn; mx = k[i] > mx ? k[i] : mx; }
    mn = warp_min(mn);
    mx = warp_max(mx);
    if (mn == mx) {
#pragma unroll
        for (int i = 0; i < kWItems; ++i)
            if ((uint32_t)(lane + 32 * i) < len) W.buf[off + lane + 32 * i] = k[i];
        __syncwarp();
        return;
    }
    uint32_t nb = 32;
    while (2 * nb < len && nb < 256) nb <<= 1;
    const uint32_t lgnb = __ffs(nb) - 1;
    const uint32_t bits = bitlen64(mx - mn);
    const uint32_t shift = bits > lgnb ? bits - lgnb : 0;
    for (uint32_t d = lane; d <= nb; d += 32) W.hist[d] = 0;
    __syncwarp();
    uint32_t rank[kWItems];
#pragma unroll
    for (int i = 0; i < kWItems; ++i)
        if ((uint32_t)(lane + 32 * i) < len) rank[i] = atomicAdd(&W.hist[(uint32_t)((k[i] - mn) >> shift)], 1u);
    __syncwarp();
    // warp exclusive scan of hist[0, nb): nb/32 contiguous entries per lane
    const uint32_t per = nb >> 5;
    uint32_t sum = 0;
    for (uint32_t j = 0; j < per; ++j) sum += W.hist[lane * per + j];
    uint32_t inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t w = __shfl_up_sync(FULL_MASK, inc, o);
        if (lane >= o) inc += w;
    }
    uint32_t run = inc - sum;
    for (uint32_t j = 0; j < per; ++j) {
        uint32_t t = W.hist[lane * per + j];
        W.hist[lane * per + j] = run;
        run += t;
    }
    if (lane == 31) W.hist[nb] = len;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < kWItems; ++i)
        if ((uint32_t)(lane + 32 * i) < len)
            W.buf[off + W.hist[(uint32_t)((k[i] - mn) >> shift)] + rank[i]] = k[i];
    __syncwarp();
    for (uint32_t d = lane; d < nb; d += 32) {
        uint32_t s0 = W.hist[d], l = W.hist[d + 1] - s0;
        if (l < 2) continue;
        if (l <= 16) insertion_sort(W.buf + off + s0, l);
        else {
            uint32_t e = atomicAdd(&W.n_stk, 1u);
            W.stk_off[e] = off + s0;
            W.stk_len[e] = l;
        }
    }
    __syncwarp();
}

__device__ void warp_sort(uint64_t (&k)[kWItems], uint32_t n, WarpSmem& W) {
    const int lane = threadIdx.x & 31;
    if (lane == 0) W.n_stk = 0;
    __syncwarp();
    warp_pass(k, 0, n, W);
    for (;;) {
        uint32_t ns = W.n_stk;
        if (ns == 0) break;
        uint32_t off = W.stk_off[ns - 1], len = W.stk_len[ns - 1];
        __syncwarp();
        if (lane == 0) W.n_stk = ns - 1;
        __syncwarp();
        if (len <= 256) {
            warp_rank_sort(W.buf + off, len);
        } else {
#pragma unroll
            for (int i = 0; i < kWItems; ++i)
                if ((uint32_t)(lane + 32 * i) < len) k[i] = W.buf[off + lane + 32 * i];
            __syncwarp();
            warp_pass(k, off, len, W);
        }
    }
}

template <bool OUT_F64>
__global__ void __launch_bounds__(kWNT) k_base_warp(const BaseItem* items, const unsigned int* count,
                                                   const uint64_t* src, void* out, Ctrl* ctrl, uint32_t list_cap) {
    extern __shared__ uint4 smem_u4[];
    WarpSmem& W = ((WarpSmem*)smem_u4)[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    if (ctrl->nan_index != ~0ull) return;
    const uint32_t ni = min(*count, list_cap);
    for (uint32_t e = blockIdx.x * kWWarps + (threadIdx.x >> 5); e < ni; e += gridDim.x * kWWarps) {
        const BaseItem it = items[e];
        const uint32_t n = (uint32_t)it.n;
        uint64_t k[kWItems];
#pragma unroll
        for (int i = 0; i < kWItems; ++i) {
            uint32_t idx = lane + 32 * i;
            if (idx < n) k[i] = __ldcs((const unsigned long long*)src + it.begin + idx);
        }
        if (n > 1) warp_sort(k, n, W);
        else if (lane == 0 && n == 1) W.buf[0] = k[0];
        __syncwarp();
        for (uint32_t idx = lane; idx < n; idx += 32) {
            uint64_t v = W.buf[idx];
            if (OUT_F64) __stcs((double*)out + it.begin + idx, decode(v));
            else __stcs((unsigned long long*)out + it.begin + idx, (unsigned long long)v);
        }
        __syncwarp();
    }
}

// --------------------------------------------------------- block base case
template <int NT, int ITEMS, int NBMAX>
struct BaseCfg {
    using BS = BlockSort<NT, ITEMS, NBMAX>;
    static constexpr size_t smem = sizeof(uint64_t) * NT * ITEMS + sizeof(typename BS::Smem);
};

template <int NT, int ITEMS, int NBMAX, bool OUT_F64>
__global__ void __launch_bounds__(NT) k_base(const BaseItem* items, const unsigned int* count, const uint64_t* src,
                                            void* out, Ctrl* ctrl, uint32_t list_cap) {
    using BS = BlockSort<NT, ITEMS, NBMAX>;
    extern __shared__ uint4 smem_u4[];
    uint64_t* a = (uint64_t*)smem_u4;
    typename BS::Smem& S = *(typename BS::Smem*)(a + NT * ITEMS);
    if (ctrl->nan_index != ~0ull) return;
    const uint32_t ni = min(*count, list_cap);
    for (uint32_t e = blockIdx.x; e < ni; e += gridDim.x) {
        const BaseItem it = items[e];
        const uint32_t n = (uint32_t)it.n;
        uint64_t k[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = threadIdx.x + i * NT;
            if (idx < n) k[i] = __ldcs((const unsigned long long*)src + it.begin + idx);
        }
        BS::sort_regs(k, a, n, S);
        __syncthreads();
        for (uint32_t idx = threadIdx.x; idx < n; idx += NT) {
            uint64_t v = a[idx];
            if (OUT_F64) __stcs((double*)out + it.begin + idx, decode(v));
            else __stcs((unsigned long long*)out + it.begin + idx, (unsigned long long)v);
        }
        __syncthreads();
    }
}

// Whole-input sort for n <= 16384 (one CTA, in place). Detects NaN first.
template <bool F64>
__global__ void __launch_bounds__(512) k_small_sort(void* keys, uint32_t n, Ctrl* ctrl) {
    using BS = BlockSort<512, 32, 8192>;
    extern __shared__ uint4 smem_u4[];
    uint64_t* a = (uint64_t*)smem_u4;
    typename BS::Smem& S = *(typename BS::Smem*)(a + 512 * 32);
    uint64_t k[32];
    uint64_t bad = ~0ull;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        uint32_t idx = threadIdx.x + i * 512;
        if (idx < n) {
            uint64_t v = ((const uint64_t*)keys)[idx];
            if (F64) {
                double d = __longlong_as_double((long long)v);
                if (isnan(d) && idx < bad) bad = idx;
                v = encode(d);
            }
            k[i] = v;
        }
    }
    if (F64) {
        bad = block_reduce_min<512>(bad, S.red);
        if (bad != ~0ull) {
            if (threadIdx.x == 0) atomicMin(&ctrl->nan_index, (unsigned long long)bad);
            return;
        }
    }
    BS::sort_regs(k, a, n, S);
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < n; idx += 512) {
        if (F64) ((double*)keys)[idx] = decode(a[idx]);
        else ((uint64_t*)keys)[idx] = a[idx];
    }
}

// --------------------------------------------------------------- fills
constexpr uint64_t kFillChunk = 1 << 16;
template <bool OUT_F64>
__global__ void __launch_bounds__(256) k_fill(const FillItem* items, const unsigned int* count, void* out,
                                             Ctrl* ctrl, uint32_t list_cap) {
    if (ctrl->nan_index != ~0ull) return;
    const uint32_t ni = min(*count, list_cap);
    uint64_t chunk0 = 0;
    for (uint32_t e = 0; e < ni; ++e) {
        const FillItem it = items[e];
        const uint64_t nch = (it.n + kFillChunk - 1) / kFillChunk;
        const uint64_t first = (blockIdx.x + gridDim.x - (chunk0 % gridDim.x)) % gridDim.x;
        const uint64_t v = OUT_F64 ? (uint64_t)__double_as_longlong(decode(it.value)) : it.value;
        for (uint64_t c = first; c < nch; c += gridDim.x) {
            uint64_t lo = it.begin + c * kFillChunk;
            uint64_t hi = min(lo + kFillChunk, it.begin + it.n);
            for (uint64_t i = lo + threadIdx.x; i < hi; i += 256) __stcs((unsigned long long*)out + i, v);
        }
        chunk0 += nch;
    }
}

// ------------------------------------------------------------- launchers
using BaseM = BaseCfg<256, 16, 4096>;
using BaseL = BaseCfg<512, 32, 8192>;

void basecase_init(int optin) {
    allow_smem(k_base_warp<true>, optin);
    allow_smem(k_base_warp<false>, optin);
    allow_smem(k_base<256, 16, 4096, true>, optin);
    allow_smem(k_base<256, 16, 4096, false>, optin);
    allow_smem(k_base<512, 32, 8192, true>, optin);
    allow_smem(k_base<512, 32, 8192, false>, optin);
    allow_smem(k_small_sort<true>, optin);
    allow_smem(k_small_sort<false>, optin);
}

void launch_base_cases(const LevelParams& p, const uint64_t* src, void* out, int out_f64, cudaStream_t st) {
    const int nsm = num_sms();
    const int gw = nsm * 5, gm = nsm * 4, gl = nsm;
    const size_t smw = sizeof(WarpSmem) * kWWarps;
    unsigned int* cnt = &p.ctrl->n_base[0];
    if (out_f64) {
        k_base_warp<true><<<gw, kWNT, smw, st>>>(p.base[0], cnt + 0, src, out, p.ctrl, p.list_cap);
        k_base<256, 16, 4096, true><<<gm, 256, BaseM::smem, st>>>(p.base[1], cnt + 1, src, out, p.ctrl, p.list_cap);
        k_base<512, 32, 8192, true><<<gl, 512, BaseL::smem, st>>>(p.base[2], cnt + 2, src, out, p.ctrl, p.list_cap);
    } else {
        k_base_warp<false><<<gw, kWNT, smw, st>>>(p.base[0], cnt + 0, src, out, p.ctrl, p.list_cap);
        k_base<256, 16, 4096, false><<<gm, 256, BaseM::smem, st>>>(p.base[1], cnt + 1, src, out, p.ctrl, p.list_cap);
        k_base<512, 32, 8192, false><<<gl, 512, BaseL::smem, st>>>(p.base[2], cnt + 2, src, out, p.ctrl, p.list_cap);
    }
}

void launch_fill(const LevelParams& p, void* out, int out_f64, int grid, cudaStream_t st) {
    if (out_f64) k_fill<true><<<grid, 256, 0, st>>>(p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
    else k_fill<false><<<grid, 256, 0, st>>>(p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
}

void launch_small_sort(void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st) {
    if (f64) k_small_sort<true><<<1, 512, BaseL::smem, st>>>(keys, (uint32_t)n, ctrl);
    else k_small_sort<false><<<1, 512, BaseL::smem, st>>>(keys, (uint32_t)n, ctrl);
}

}  // namespace lsort_dev
