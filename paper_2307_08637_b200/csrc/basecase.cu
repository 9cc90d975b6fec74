// basecase.cu -- small-segment sorts and equality fills.
//
//   k_base_smem / k_base_reg
//                 one CTA per segment, three size classes: 128 threads for
//                 <= 1024 keys (TMA into shared memory), 256 for <= 4096 and
//                 1024 for <= 16384 (keys in registers): range-adaptive
//                 counting pass + collision fix-up (SmemSort), decode on store.
//   k_small_sort  whole inputs of <= 16384 keys, in place, NaN check first.
//   k_fill        equality buckets / homogeneous segments: value stores only.
// Together they replace radix_base_case_sort + insertion sort
// and mark_homogeneous.
#include <algorithm>

#include "kernels_common.cuh"
#include "smemsort.cuh"
#include "tma.cuh"

namespace lsort_dev {

template <int NT, int CAP, int NBMAX, bool OUT_F64>
__global__ void __launch_bounds__(NT) k_base_smem(const BaseItem* items, const unsigned int* count, const uint64_t* src,
                                                 void* out, Ctrl* ctrl, uint32_t list_cap) {
    griddep_wait();
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
        const uint64_t* g = src + it.rd;
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
        const uint64_t* res = a;
        if (n > 1) {
            SS::sort_fast(a, n, S);
            res = S.B;
        }
        for (uint32_t i = threadIdx.x; i < n; i += NT) {
            const uint64_t v = res[i];
            if (OUT_F64) __stcs((double*)out + it.begin + i, decode(v));
            else __stcs((unsigned long long*)out + it.begin + i, (unsigned long long)v);
        }
        __syncthreads();
    }
}

// Keys read straight into registers (coalesced 8-byte loads, no staging
// array): shared memory holds only the output array + digit histogram, so
// three CTAs share an SM and hide each other's load latency. The segment's
// own input range doubles as scratch for the rare large-digit passes.
template <int IT, class SS, bool OUT_F64>
__device__ __forceinline__ void base_reg_one(uint64_t* g, uint32_t n, typename SS::SmemR& S, void* out,
                                             uint64_t begin) {
    constexpr int NT = SS::kThreads;
    uint64_t k[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const uint32_t j = threadIdx.x + i * NT;
        k[i] = j < n ? __ldcs((const unsigned long long*)g + j) : 0ull;
    }
    SS::sort_regs(k, n, S, g);
    for (uint32_t i = threadIdx.x; i < n; i += NT) {
        const uint64_t v = S.B[i];
        if (OUT_F64) __stcs((double*)out + begin + i, decode(v));
        else __stcs((unsigned long long*)out + begin + i, (unsigned long long)v);
    }
}

// Keys read straight into registers (coalesced 8-byte loads, no staging
// array): shared memory holds only the output array + digit histogram, so
// three CTAs share an SM and hide each other's load latency. The segment's
// own input range doubles as scratch for the rare large-digit passes.
// Segments of at most CAP / 2 keys take a half-width register array so no
// thread issues work for slots past n.
// nmin < n <= nmax: the items of the list this kernel takes (one list may be
// shared by two kernels of different CTA shapes, split by segment size).
template <int NT, int CAP, int NBMAX, int MINB, bool OUT_F64>
__global__ void __launch_bounds__(NT, MINB) k_base_reg(const BaseItem* items, const unsigned int* count, uint64_t* src,
                                                   void* out, Ctrl* ctrl, uint32_t list_cap, uint32_t nmin,
                                                   uint32_t nmax) {
    griddep_wait();
    using SS = SmemSort<NT, CAP, NBMAX>;
    extern __shared__ uint4 smem_u4[];
    typename SS::SmemR& S = *(typename SS::SmemR*)smem_u4;
    if (ctrl->nan_index != ~0ull) return;
    const uint32_t ni = min(*count, list_cap);
    // the next segment of this CTA is pulled into L2 while this one sorts
    // (its register loads then wait on L2, not HBM, latency)
    if (threadIdx.x == 0 && blockIdx.x < ni) l2_prefetch(src + items[blockIdx.x].rd, 8 * items[blockIdx.x].n);
    for (uint32_t e = blockIdx.x; e < ni; e += gridDim.x) {
        const BaseItem it = items[e];
        const uint32_t n = (uint32_t)it.n;
        if (n <= nmin || n > nmax) continue;
        uint64_t* g = src + it.rd;
        if (threadIdx.x == 0 && e + gridDim.x < ni) {
            const BaseItem nx = items[e + gridDim.x];
            if (nx.n > nmin && nx.n <= nmax) l2_prefetch(src + nx.rd, 8 * nx.n);
        }
        // register array of 1/2, 3/4 or all of CAP / NT keys per thread: every
        // unused slot still issues its predicated loads, digit, rank and placement
        if (n <= (uint32_t)CAP / 2) base_reg_one<SS::ITEMS / 2, SS, OUT_F64>(g, n, S, out, it.begin);
        else if (n <= (uint32_t)CAP / 4 * 3) base_reg_one<SS::ITEMS / 4 * 3, SS, OUT_F64>(g, n, S, out, it.begin);
        else base_reg_one<SS::ITEMS, SS, OUT_F64>(g, n, S, out, it.begin);
        // no barrier: the next segment writes shared memory (hist, reduction
        // words) that the output loop does not read, and S.B only after its
        // first barrier
    }
}

// --------------------------------------------------------- block base case
template <int NT, int ITEMS, int NBMAX>
struct BaseCfg {
    using BS = BlockSort<NT, ITEMS, NBMAX>;
    static constexpr size_t smem = sizeof(uint64_t) * NT * ITEMS + sizeof(typename BS::Smem);
};

// Whole-input sort for n <= 16384 (one CTA, in place). Detects NaN first.
template <bool F64>
__global__ void __launch_bounds__(1024) k_small_sort(void* keys, uint32_t n, Ctrl* ctrl) {
    griddep_wait();
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
constexpr uint64_t kFillChunk = 1 << 14;
// Equality fills: CTA (x, y) of a (G, kFillSplit) grid takes items x, x+G, ...
// and within an item the chunks y, y+kFillSplit, ... -- no CTA walks the whole
// item list, and large items still spread over kFillSplit CTAs.
constexpr uint32_t kFillSplit = 8;
template <bool OUT_F64>
__global__ void __launch_bounds__(256) k_fill(const FillItem* items, const unsigned int* count, void* out,
                                             Ctrl* ctrl, uint32_t list_cap) {
    griddep_wait();
    if (ctrl->nan_index != ~0ull) return;
    const uint32_t ni = min(*count, list_cap);
    for (uint32_t e = blockIdx.x; e < ni; e += gridDim.x) {
        const FillItem it = items[e];
        const uint64_t v = OUT_F64 ? (uint64_t)__double_as_longlong(decode(it.value)) : it.value;
        const uint64_t nch = (it.n + kFillChunk - 1) / kFillChunk;
        for (uint64_t c = blockIdx.y; c < nch; c += gridDim.y) {
            const uint64_t lo = it.begin + c * kFillChunk;
            const uint64_t hi = min(lo + kFillChunk, it.begin + it.n);
            for (uint64_t i = lo + threadIdx.x; i < hi; i += 256) __stcs((unsigned long long*)out + i, v);
        }
    }
}

// ------------------------------------------------------------- launchers
// size classes: <= 1024 keys in shared memory (TMA), <= 4096 and <= 16384 in registers
using SmallSS = SmemSort<128, 1024, 1024>;
using BaseL = BaseCfg<1024, 16, 8192>;
static_assert(1024 == kWarpBaseCap, "small base-case class");

template <int NT, int CAP, int NBMAX, int MINB>
static void reg_init(int optin) {
    allow_smem(k_base_reg<NT, CAP, NBMAX, MINB, true>, optin);
    allow_smem(k_base_reg<NT, CAP, NBMAX, MINB, false>, optin);
}

void basecase_init(int optin) {
    allow_smem(k_base_smem<128, 1024, 1024, true>, optin);
    allow_smem(k_base_smem<128, 1024, 1024, false>, optin);
    reg_init<256, 4096, 4096, 4>(optin);
    reg_init<512, 8192, 4096, 2>(optin);
    reg_init<1024, 16384, 8192, 1>(optin);
    allow_smem(k_small_sort<true>, optin);
    allow_smem(k_small_sort<false>, optin);
}

template <int NT, int CAP, int NBMAX, int MINB>
static void launch_reg(const LevelParams& p, int cls, const uint64_t* src, void* out, int out_f64, cudaStream_t st,
                       uint32_t nmin, uint32_t nmax) {
    const size_t sm = sizeof(typename SmemSort<NT, CAP, NBMAX>::SmemR);
    const int grid = num_sms() * MINB;
    unsigned int* cnt = &p.ctrl->n_base[cls];
    if (out_f64)
        pdl(k_base_reg<NT, CAP, NBMAX, MINB, true>, grid, NT, sm, st, p.base[cls], cnt, (uint64_t*)src, out, p.ctrl,
            p.list_cap, nmin, nmax);
    else
        pdl(k_base_reg<NT, CAP, NBMAX, MINB, false>, grid, NT, sm, st, p.base[cls], cnt, (uint64_t*)src, out, p.ctrl,
            p.list_cap, nmin, nmax);
}

// One size class on its own stream: 0 (<= 1 Ki keys, shared memory), 1 (<= 4 Ki),
// and the 16 Ki list split by size into 3 (<= 8 Ki keys: 512 threads, two
// CTAs per SM) and 2 (> 8 Ki: 1024 threads, one CTA per SM) -- a single
// 1024-thread class cost 1.5x the 4 Ki class per key (one segment per SM,
// no overlap); the classes are independent, so they run side by side.
void launch_base_class(const LevelParams& p, int cls, const uint64_t* src, void* out, int out_f64, cudaStream_t st) {
    const int nsm = num_sms();
    if (cls == 0) {
        unsigned int* cnt = &p.ctrl->n_base[0];
        const size_t sm = sizeof(SmallSS::Smem);
        if (out_f64) pdl(k_base_smem<128, 1024, 1024, true>, nsm * 8, 128, sm, st, p.base[0], cnt, src, out, p.ctrl, p.list_cap);
        else pdl(k_base_smem<128, 1024, 1024, false>, nsm * 8, 128, sm, st, p.base[0], cnt, src, out, p.ctrl, p.list_cap);
    } else if (cls == 1) {
        launch_reg<256, 4096, 4096, 4>(p, 1, src, out, out_f64, st, 0, 4096);
    } else if (cls == 2) {
        launch_reg<1024, 16384, 8192, 1>(p, 2, src, out, out_f64, st, 8192, 16384);
    } else {
        launch_reg<512, 8192, 4096, 2>(p, 2, src, out, out_f64, st, 0, 8192);
    }
}

void launch_base_cases(const LevelParams& p, const uint64_t* src, void* out, int out_f64, cudaStream_t st) {
    for (int c = 0; c < kBaseLaunches; ++c) launch_base_class(p, c, src, out, out_f64, st);
}

void launch_fill(const LevelParams& p, void* out, int out_f64, int grid, cudaStream_t st) {
    const dim3 g((unsigned)grid, kFillSplit);
    if (out_f64) pdl(k_fill<true>, g, 256, 0, st, p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
    else pdl(k_fill<false>, g, 256, 0, st, p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
}

void launch_small_sort(void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st) {
    if (f64) pdl(k_small_sort<true>, 1, 1024, BaseL::smem, st, keys, (uint32_t)n, ctrl);
    else pdl(k_small_sort<false>, 1, 1024, BaseL::smem, st, keys, (uint32_t)n, ctrl);
}

}  // namespace lsort_dev
