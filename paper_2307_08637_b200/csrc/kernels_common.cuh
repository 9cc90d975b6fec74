// kernels_common.cuh -- device helpers shared by the partition, model,
// base-case and utility kernels.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace lsort_dev {

#define FULL_MASK 0xffffffffu

__device__ __forceinline__ uint64_t load_key(const void* src, uint64_t i, bool f64) {
    uint64_t v = ((const uint64_t*)src)[i];
    return f64 ? encode(__longlong_as_double((long long)v)) : v;
}

// Per-segment sampling stream (same definition as oracle lso_seg_seed).
__device__ __forceinline__ uint64_t seg_seed(uint64_t cfg_seed, uint64_t begin, uint32_t depth) {
    return splitmix64(cfg_seed ^ splitmix64(begin + ((uint64_t)depth << 48)));
}
// SPEC.md:438 (same double arithmetic as oracle lso_first_sample_size)
__device__ __forceinline__ uint64_t first_sample_size(const DevCfg& c, uint64_t n) {
    double v = __dmul_rn(c.sample_fraction, __ull2double_rn(n));
    double cap = (double)c.first_sample_cap;
    uint64_t s = (uint64_t)ceil(v < cap ? v : cap);
    return s < 2 ? 2 : s;
}
__device__ __forceinline__ uint64_t rmi_sample_size(const DevCfg& c, uint64_t n) {
    double v = __dmul_rn(c.sample_fraction, __ull2double_rn(n));
    double cap = (double)c.rmi_sample_cap;
    uint64_t s = (uint64_t)ceil(v < cap ? v : cap);
    return s < 2 ? 2 : s;
}

__device__ __forceinline__ uint32_t model_payload_bytes(const ModelHdr& h) {
    if (h.kind == kLearned) return kLearnedEntryBytes * h.B;
    if (h.kind == kTree) return (uint32_t)((tree_payload_bytes(h.leaf_origin, h.nsplit) + 15) & ~15ull);
    if (h.kind == kRadix && (h.flags & kModelLog)) return ((2 * h.levels + 15) & ~15u) + ((2 * h.B + 15) & ~15u);
    if (h.kind == kRadix && (h.flags & kModelLut)) return (2 * h.B + 15) & ~15u;
    return 0;
}

// Copy a model record (header + payload) into shared memory.
__device__ __forceinline__ void load_model_smem(const uint8_t* g, uint8_t* s) {
    const uint4* gs = (const uint4*)g;
    uint4* ss = (uint4*)s;
    if (threadIdx.x < 8) ss[threadIdx.x] = gs[threadIdx.x];
    __syncthreads();
    uint32_t words = model_payload_bytes(*(const ModelHdr*)s) / 16;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) ss[8 + i] = gs[8 + i];
    __syncthreads();
}

struct MView {
    const ModelHdr* h;
    const RmiEntry* e;
    const uint64_t* tree;
    const uint64_t* spl;
    const uint32_t* eqo;
};
__device__ __forceinline__ MView model_view(const uint8_t* s) {
    MView m;
    m.h = (const ModelHdr*)s;
    const uint8_t* p = s + sizeof(ModelHdr);
    m.e = (const RmiEntry*)p;
    m.tree = (const uint64_t*)p;
    m.spl = m.tree + m.h->leaf_origin;
    m.eqo = (const uint32_t*)(m.spl + m.h->nsplit);
    return m;
}

// Generic classifier over a model copied to shared memory (unit-test and
// multi-GPU paths; the hot partition kernels use per-kind specialisations).
struct Classifier {
    uint32_t kind, nb, B, levels, leaf_origin, nsplit, shift, flags;
    double rs, ri, base, scale, cdf_lo, inv_span;
    uint64_t rmin;
    MView m;
    __device__ __forceinline__ void init(const uint8_t* s) {
        m = model_view(s);
        const ModelHdr& h = *m.h;
        kind = h.kind; nb = h.nbuckets; B = h.B; levels = h.levels; leaf_origin = h.leaf_origin;
        nsplit = h.nsplit; shift = h.shift; flags = h.flags; rs = h.root_slope; ri = h.root_icpt; base = h.key_base;
        scale = h.key_scale; cdf_lo = h.cdf_lo; inv_span = h.inv_span; rmin = h.radix_min;
    }
    template <uint32_t KIND>
    __device__ __forceinline__ uint32_t classify(uint64_t x) const {
        if constexpr (KIND == kLearned) {
            double xn = rmi_normalize(base, scale, x);
            const RmiEntry s = m.e[rmi_route(rs, ri, B, xn)];
            return cdf_bucket_clamped(clamp_pred(__dadd_rn(__dmul_rn(s.slope, xn), s.intercept), s.lo, s.hi),
                                      cdf_lo, inv_span, nb);
        } else if constexpr (KIND == kTree) {
            return tree_bucket(levels, leaf_origin, nsplit, m.tree, m.spl, m.eqo, x);
        } else if constexpr (KIND == kRadix) {
            if (flags & kModelLog) {
                const uint16_t* tab = (const uint16_t*)(m.h + 1);
                const uint16_t* lut = tab + ((levels + 7) & ~7u);
                return lut[binade_cell(x, tab, (uint32_t)rmin, levels, B)];
            }
            if (flags & kModelLut) return ((const uint16_t*)(m.h + 1))[lut_cell(x, rmin, shift, B)];
            uint64_t d = (x - rmin) >> shift;
            return d >= nb ? nb - 1 : (uint32_t)d;
        } else {
            return 0u | (1u << 31);
        }
    }
    __device__ __forceinline__ uint32_t classify_any(uint64_t x) const {
        switch (kind) {
        case kLearned: return classify<kLearned>(x);
        case kTree: return classify<kTree>(x);
        case kRadix: return classify<kRadix>(x);
        default: return classify<kFill>(x);
        }
    }
};

// Shared-memory histogram add. Measured on B200 (tools/micro/hist_bench.cu,
// profiles/): a plain shared atomicAdd runs at full HBM rate for spread and
// for all-equal bins (the hardware aggregates same-address lanes), while
// __match_any_sync warp aggregation is ADU-bound and 6.5x slower for spread
// bins -- so aggregation is left to the hardware here.
__device__ __forceinline__ void hist_add(uint32_t* hist, uint32_t b, bool valid) {
    if (valid) atomicAdd(&hist[b], 1u);
}
// Rank of this lane's key within its bucket (all lanes must call). Returning
// atomics serialise on equal addresses (3x slower when a warp shares one
// bucket), so a warp-uniform bucket takes one atomic for the whole warp.
__device__ __forceinline__ uint32_t hist_rank_warp(uint32_t* hist, uint32_t b, bool valid) {
    const unsigned vmask = __ballot_sync(FULL_MASK, valid);
    const int lane = threadIdx.x & 31;
    const int first = __ffs(vmask) - 1;
    const uint32_t b0 = __shfl_sync(FULL_MASK, b, first < 0 ? 0 : first);
    if (__all_sync(FULL_MASK, !valid || b == b0)) {
        uint32_t old = 0;
        if (lane == first) old = atomicAdd(&hist[b0], (uint32_t)__popc(vmask));
        old = __shfl_sync(FULL_MASK, old, first < 0 ? 0 : first);
        return old + __popc(vmask & ((1u << lane) - 1u));
    }
    return valid ? atomicAdd(&hist[b], 1u) : 0u;
}

// last s in [0,n) with prefix[s] <= tile
__device__ __forceinline__ uint32_t find_seg(const uint64_t* prefix, uint32_t nsegs, uint64_t tile) {
    uint32_t lo = 0, hi = nsegs;
    while (hi - lo > 1) {
        uint32_t mid = (lo + hi) >> 1;
        if (prefix[mid] <= tile) lo = mid; else hi = mid;
    }
    return lo;
}

// Tile geometry: keys [lo,hi) read as 16-byte pairs over the 16-byte aligned
// interior plus at most two single keys (head / tail).
struct TileGeom {
    uint64_t lo, hi, a0;
    uint32_t npairs;
    uint32_t nsingle;
    uint64_t s0, s1;  // head / tail single (scalars: an indexed array would live in local memory)
    __device__ __forceinline__ void init(const void* base, uint64_t l, uint64_t h) {
        lo = l; hi = h;
        uint64_t par = (((uintptr_t)base) >> 3) & 1;
        a0 = lo + ((lo + par) & 1);
        if (a0 > hi) a0 = hi;
        npairs = (uint32_t)((hi - a0) / 2);
        const uint64_t t = a0 + 2ull * npairs;
        const bool head = a0 > lo, tail = t < hi;
        nsingle = (uint32_t)head + (uint32_t)tail;
        s0 = head ? lo : t;
        s1 = t;
    }
    __device__ __forceinline__ uint64_t single(uint32_t i) const { return i == 0 ? s0 : s1; }
};

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialisation (pdl() below) and waits here for its predecessor's
// results -- the next kernel's launch overlaps the previous kernel's tail
// instead of a full launch gap after it (the sort is a chain of ~40 kernels).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();  // false when LSORT_NO_PDL is set (A/B measurement)
template <typename... KArgs, typename... Args>
inline void pdl(void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t c = {};
    c.gridDim = g;
    c.blockDim = b;
    c.dynamicSmemBytes = sm;
    c.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    c.attrs = a;
    c.numAttrs = 1;
    cudaLaunchKernelEx(&c, k, args...);
    // LSORT_SYNC_DEBUG: synchronise after every launch and name the first kernel that
    // faults (compute-sanitizer stand-in; never set in a measured run)
    static const bool sync_debug = getenv("LSORT_SYNC_DEBUG") != nullptr;
    if (sync_debug) {
        const cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            const char* name = nullptr;
            cudaFuncGetName(&name, (const void*)k);
            fprintf(stderr, "[lsort sync-debug] %s after kernel %s grid %u block %u\n", cudaGetErrorString(e),
                    name ? name : __PRETTY_FUNCTION__, g.x, b.x);
            abort();
        }
    }
}

template <class F>
inline void allow_smem(F* f, int optin) {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, f) != cudaSuccess) { cudaGetLastError(); return; }
    int dyn = optin - (int)a.sharedSizeBytes;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess) cudaGetLastError();
}

}  // namespace lsort_dev
