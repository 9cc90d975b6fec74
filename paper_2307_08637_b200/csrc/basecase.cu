// basecase.cu -- small-segment sorts and equality fills.
//
//   k_base        one CTA per segment, three size classes: 64 threads for
//                 <= 512 keys, 256 for <= 4096, 1024 for <= 16384 (BlockSort:
//                 range-adaptive counting pass + rank-within-digit placement),
//                 decode on store.
//   k_small_sort  whole inputs of <= 16384 keys, in place, NaN check first.
//   k_fill        equality buckets / homogeneous segments: value stores only.
// Together they replace radix_base_case_sort + insertion sort
// and mark_homogeneous.
#include <algorithm>

#include "kernels_common.cuh"
#include "tma.cuh"

namespace lsort_dev {

// ------------------------------------------------ shared-memory base case
// Segment sort that lives in shared memory: TMA bulk load (cp.async.bulk +
// mbarrier) of the segment, then the BlockSort algorithm with rolled loops
// over shared arrays (A keys, B staging, R 16-bit ranks) instead of unrolled
// register arrays: a range-adaptive counting pass, rank-within-digit
// placement for digits <= 16 keys, warp rank sort for <= 256, another pass
// for larger digits. Decode fused into the coalesced store.
template <int NT, int CAP, int NBMAX>
struct SmemSort {
    static constexpr int kSmall = 16;
    static constexpr int kMedium = 256;
    static constexpr int kStk = CAP / (kSmall + 1) + 2;
    static_assert(CAP <= 65536, "16-bit ranks");
    struct Smem {
        uint64_t A[CAP + 4];  // logical key i at A[mis + i]
        uint64_t B[CAP];
        uint32_t hist[NBMAX + 1];
        uint16_t R[CAP];
        uint32_t wsum[NT / 32 + 1];
        uint64_t red[2 * (NT / 32)];
        uint32_t n_med, n_large;
        uint32_t med_off[kStk], med_len[kStk], large_off[kStk], large_len[kStk];
        uint64_t mbar;
    };

    __device__ static __forceinline__ void push(Smem& S, uint32_t at, uint32_t l) {
        if (l <= (uint32_t)kMedium) {
            uint32_t q = atomicAdd(&S.n_med, 1u);
            S.med_off[q] = at;
            S.med_len[q] = l;
        } else {
            uint32_t q = atomicAdd(&S.n_large, 1u);
            S.large_off[q] = at;
            S.large_len[q] = l;
        }
    }

    // one distribution pass over a[off, off+len), staging through b
    __device__ static void pass(uint64_t* a, uint64_t* b, uint32_t off, uint32_t len, Smem& S) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        uint64_t mn = ~0ull, mx = 0;
        for (uint32_t i = tid; i < len; i += NT) {
            uint64_t k = a[off + i];
            mn = k < mn ? k : mn;
            mx = k > mx ? k : mx;
        }
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t a1 = __shfl_xor_sync(FULL_MASK, mn, o), b1 = __shfl_xor_sync(FULL_MASK, mx, o);
            mn = a1 < mn ? a1 : mn;
            mx = b1 > mx ? b1 : mx;
        }
        __syncthreads();  // previous users of red / hist are done
        if (lane == 0) { S.red[2 * warp] = mn; S.red[2 * warp + 1] = mx; }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            uint64_t a1 = S.red[2 * w], b1 = S.red[2 * w + 1];
            mn = a1 < mn ? a1 : mn;
            mx = b1 > mx ? b1 : mx;
        }
        if (mn == mx) return;  // homogeneous range: already sorted
        uint32_t nb = 1;
        while (2 * nb < len && nb < (uint32_t)NBMAX) nb <<= 1;
        const uint32_t lgnb = __ffs(nb) - 1;
        const uint32_t bits = bitlen64(mx - mn);
        const uint32_t shift = bits > lgnb ? bits - lgnb : 0;
        for (uint32_t d = tid; d < nb; d += NT) S.hist[d] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < len; i += NT)
            S.R[off + i] = (uint16_t)atomicAdd(&S.hist[(uint32_t)((a[off + i] - mn) >> shift)], 1u);
        __syncthreads();
        {  // exclusive scan with big-digit detection
            const uint32_t per = (nb + NT - 1) / NT;
            const uint32_t lo = min(nb, tid * per), hi = min(nb, lo + per);
            uint32_t sum = 0;
            for (uint32_t d = lo; d < hi; ++d) sum += S.hist[d];
            uint32_t incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t w = __shfl_up_sync(FULL_MASK, incl, o);
                if (lane >= o) incl += w;
            }
            if (lane == 31) S.wsum[warp] = incl;
            __syncthreads();
            uint32_t run = incl - sum;
            for (int w = 0; w < warp; ++w) run += S.wsum[w];
            for (uint32_t d = lo; d < hi; ++d) {
                uint32_t t = S.hist[d];
                S.hist[d] = run;
                if (t > (uint32_t)kSmall) push(S, off + run, t);
                run += t;
            }
            if (tid == 0) S.hist[nb] = len;
        }
        __syncthreads();
        for (uint32_t i = tid; i < len; i += NT) {
            const uint64_t k = a[off + i];
            b[off + S.hist[(uint32_t)((k - mn) >> shift)] + S.R[off + i]] = k;
        }
        __syncthreads();
        for (uint32_t j = tid; j < len; j += NT) {
            const uint64_t k = b[off + j];
            const uint32_t d = (uint32_t)((k - mn) >> shift);
            const uint32_t s0 = S.hist[d], c = S.hist[d + 1] - s0;
            uint32_t p = j;
            if (c <= (uint32_t)kSmall) {
                p = s0;
                for (uint32_t t = s0; t < s0 + c; ++t) {
                    const uint64_t w = b[off + t];
                    p += (w < k) || (w == k && t < j);
                }
            }
            a[off + p] = k;
        }
        __syncthreads();
    }

    __device__ static void warp_rank_sort(uint64_t* a, uint32_t len) {
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

    // sort a[0,n) (keys already in shared memory)
    __device__ static void sort(uint64_t* a, uint32_t n, Smem& S) {
        if (threadIdx.x == 0) { S.n_med = 0; S.n_large = 0; }
        __syncthreads();
        pass(a, S.B, 0, n, S);
        __syncthreads();
        const int warp = threadIdx.x >> 5;
        for (;;) {
            const uint32_t nm = S.n_med, nl = S.n_large;
            if (nm == 0 && nl == 0) break;
            for (uint32_t e = warp; e < nm; e += NT / 32) warp_rank_sort(a + S.med_off[e], S.med_len[e]);
            __syncthreads();
            if (threadIdx.x == 0) S.n_med = 0;
            if (nl == 0) { __syncthreads(); break; }
            const uint32_t off = S.large_off[nl - 1], len = S.large_len[nl - 1];
            __syncthreads();
            if (threadIdx.x == 0) S.n_large = nl - 1;
            pass(a, S.B, off, len, S);
            __syncthreads();
        }
    }
};

template <int NT, int CAP, int NBMAX, bool OUT_F64>
__global__ void __launch_bounds__(NT) k_base_smem(const BaseItem* items, const unsigned int* count, const uint64_t* src,
                                                 void* out, Ctrl* ctrl, uint32_t list_cap) {
    using SS = SmemSort<NT, CAP, NBMAX>;
    extern __shared__ uint4 smem_u4[];
    typename SS::Smem& S = *(typename SS::Smem*)smem_u4;
    if (ctrl->nan_index != ~0ull) return;
    const uint32_t ni = min(*count, list_cap);
    if (threadIdx.x == 0) mbar_init(&S.mbar, 1);
    __syncthreads();
    uint32_t phase = 0;
    for (uint32_t e = blockIdx.x; e < ni; e += gridDim.x) {
        const BaseItem it = items[e];
        const uint32_t n = (uint32_t)it.n;
        const uint64_t* g = src + it.begin;
        // TMA bulk load of the 16-byte aligned interior; head/tail keys by threads
        const uint32_t mis = (uint32_t)(((uintptr_t)g >> 3) & 1);
        const uint32_t head = min(mis, n);
        const uint32_t body = (n - head) & ~1u;
        uint64_t* a = S.A + mis;
        if (threadIdx.x == 0 && body) {
            mbar_expect_tx(&S.mbar, body * 8);
            tma_load_1d(a + head, g + head, body * 8, &S.mbar);
        }
        if (threadIdx.x == 32 && head) a[0] = g[0];
        if (threadIdx.x == 64 && head + body < n) a[n - 1] = g[n - 1];
        if (body) mbar_wait(&S.mbar, phase);
        phase ^= (body ? 1u : 0u);
        __syncthreads();
        if (n > 1) SS::sort(a, n, S);
        for (uint32_t i = threadIdx.x; i < n; i += NT) {
            const uint64_t v = a[i];
            if (OUT_F64) __stcs((double*)out + it.begin + i, decode(v));
            else __stcs((unsigned long long*)out + it.begin + i, (unsigned long long)v);
        }
        __syncthreads();
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
__global__ void __launch_bounds__(1024) k_small_sort(void* keys, uint32_t n, Ctrl* ctrl) {
    using BS = BlockSort<1024, 16, 8192>;
    extern __shared__ uint4 smem_u4[];
    uint64_t* a = (uint64_t*)smem_u4;
    typename BS::Smem& S = *(typename BS::Smem*)(a + 1024 * 16);
    uint64_t k[16];
    uint64_t bad = ~0ull;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        uint32_t idx = threadIdx.x + i * 1024;
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
        bad = block_reduce_min<1024>(bad, S.red);
        if (bad != ~0ull) {
            if (threadIdx.x == 0) atomicMin(&ctrl->nan_index, (unsigned long long)bad);
            return;
        }
    }
    BS::sort_regs(k, a, n, S);
    __syncthreads();
    for (uint32_t idx = threadIdx.x; idx < n; idx += 1024) {
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
// size classes: <= 1024 and <= 4096 keys in shared memory (TMA), <= 16384 in registers
using SmallSS = SmemSort<128, 1024, 512>;
using MidSS = SmemSort<512, 4096, 2048>;
using BaseL = BaseCfg<1024, 16, 8192>;
static_assert(1024 == kWarpBaseCap, "small base-case class");

void basecase_init(int optin) {
    allow_smem(k_base_smem<128, 1024, 512, true>, optin);
    allow_smem(k_base_smem<128, 1024, 512, false>, optin);
    allow_smem(k_base_smem<512, 4096, 2048, true>, optin);
    allow_smem(k_base_smem<512, 4096, 2048, false>, optin);
    allow_smem(k_base<1024, 16, 8192, true>, optin);
    allow_smem(k_base<1024, 16, 8192, false>, optin);
    allow_smem(k_small_sort<true>, optin);
    allow_smem(k_small_sort<false>, optin);
}

void launch_base_cases(const LevelParams& p, const uint64_t* src, void* out, int out_f64, cudaStream_t st) {
    const int nsm = num_sms();
    const int g0 = nsm * 8, g1 = nsm * 2, gl = nsm;
    const size_t s0 = sizeof(SmallSS::Smem), s1 = sizeof(MidSS::Smem);
    unsigned int* cnt = &p.ctrl->n_base[0];
    if (out_f64) {
        k_base_smem<128, 1024, 512, true><<<g0, 128, s0, st>>>(p.base[0], cnt + 0, src, out, p.ctrl, p.list_cap);
        k_base_smem<512, 4096, 2048, true><<<g1, 512, s1, st>>>(p.base[1], cnt + 1, src, out, p.ctrl, p.list_cap);
        k_base<1024, 16, 8192, true><<<gl, 1024, BaseL::smem, st>>>(p.base[2], cnt + 2, src, out, p.ctrl, p.list_cap);
    } else {
        k_base_smem<128, 1024, 512, false><<<g0, 128, s0, st>>>(p.base[0], cnt + 0, src, out, p.ctrl, p.list_cap);
        k_base_smem<512, 4096, 2048, false><<<g1, 512, s1, st>>>(p.base[1], cnt + 1, src, out, p.ctrl, p.list_cap);
        k_base<1024, 16, 8192, false><<<gl, 1024, BaseL::smem, st>>>(p.base[2], cnt + 2, src, out, p.ctrl, p.list_cap);
    }
}

void launch_fill(const LevelParams& p, void* out, int out_f64, int grid, cudaStream_t st) {
    if (out_f64) k_fill<true><<<grid, 256, 0, st>>>(p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
    else k_fill<false><<<grid, 256, 0, st>>>(p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
}

void launch_small_sort(void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st) {
    if (f64) k_small_sort<true><<<1, 1024, BaseL::smem, st>>>(keys, (uint32_t)n, ctrl);
    else k_small_sort<false><<<1, 1024, BaseL::smem, st>>>(keys, (uint32_t)n, ctrl);
}

}  // namespace lsort_dev
