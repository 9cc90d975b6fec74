// kernels.cu -- sm_100a kernels of the B200 LearnedSort (AIPS2o) hot path.
//
//   k_build_models   Alg. 5 policy per segment: device-drawn samples, shared-
//                    memory sample sort, duplicate fraction, then RMI training
//                    (fit_line/Rmi::train/enforce_monotonic, models.cpp:14-131)
//                    or SplitterTree::build (models.cpp:133-185) -- one CTA per
//                    segment.
//   k_classify_hist  fused encode + model inference + warp-aggregated shared-
//                    memory histogram (classification half of classify_and_flush,
//                    SPEC.md:311-319), 128-bit loads, persistent over tiles.
//   k_scan_children  per-segment exclusive scan of bucket counts -> write
//                    cursors; emits base-case / equality-fill / recursion work
//                    (boundary computation + mark_homogeneous).
//   k_scatter        re-classify, claim per-bucket ranges, stage the tile in
//                    shared memory grouped by bucket, write coalesced runs
//                    (flush + permute of SPEC.md:311-328, out of place).
//   k_base           shared-memory MSD block sort of small segments, decode on
//                    store (radix_base_case_sort).
//   k_fill           equality buckets / homogeneous segments.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "kernels.cuh"

namespace lsort_dev {

#define FULL_MASK 0xffffffffu

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ uint64_t load_key(const void* src, uint64_t i, bool f64) {
    uint64_t v = ((const uint64_t*)src)[i];
    return f64 ? encode(__longlong_as_double((long long)v)) : v;
}

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
    if (h.kind == kLearned) return 32u * h.B;
    if (h.kind == kTree) return (uint32_t)((tree_payload_bytes(h.leaf_origin, h.nsplit) + 15) & ~15ull);
    return 0;
}

// Copy a model record (header + payload) into shared memory.
__device__ void load_model_smem(const uint8_t* g, uint8_t* s) {
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

// Per-key classifier for a model held in shared memory. Returns the bucket
// id with bit 31 set for keys of an equality bucket (value known, no move).
struct Classifier {
    uint32_t kind, nb, B, levels, leaf_origin, nsplit, shift;
    double rs, ri, base, scale, cdf_lo, inv_span;
    uint64_t rmin;
    MView m;
    __device__ __forceinline__ void init(const uint8_t* s) {
        m = model_view(s);
        const ModelHdr& h = *m.h;
        kind = h.kind; nb = h.nbuckets; B = h.B; levels = h.levels; leaf_origin = h.leaf_origin;
        nsplit = h.nsplit; shift = h.shift; rs = h.root_slope; ri = h.root_icpt; base = h.key_base;
        scale = h.key_scale; cdf_lo = h.cdf_lo; inv_span = h.inv_span; rmin = h.radix_min;
    }
    template <uint32_t KIND>
    __device__ __forceinline__ uint32_t classify(uint64_t x) const {
        if constexpr (KIND == kLearned) {
            // models.hpp:34-43 + 162-171, bit-exact (no FMA contraction)
            double xn = rmi_normalize(base, scale, x);
            uint32_t i = rmi_route(rs, ri, B, xn);
            const RmiEntry s = m.e[i];
            double v = __dadd_rn(__dmul_rn(s.slope, xn), s.intercept);
            if (v < s.lo) v = s.lo;
            if (v > s.hi) v = s.hi;
            if (v < 0.0) v = 0.0;
            if (v > 1.0) v = 1.0;
            double t = __dmul_rn(__dmul_rn(__dsub_rn(v, cdf_lo), inv_span), (double)nb);
            if (!(t > 0.0)) return 0;
            if (t >= (double)nb) return nb - 1;
            return (uint32_t)t;
        } else if constexpr (KIND == kTree) {
            return tree_bucket(levels, leaf_origin, nsplit, m.tree, m.spl, m.eqo, x);
        } else if constexpr (KIND == kRadix) {
            uint64_t d = (x - rmin) >> shift;
            return d >= nb ? nb - 1 : (uint32_t)d;
        } else {
            return 0u | (1u << 31);  // kFill: everything equal
        }
    }
};

// warp-aggregated shared-memory histogram add (all lanes must call)
__device__ __forceinline__ void hist_add_warp(uint32_t* hist, uint32_t b, bool valid) {
    unsigned vmask = __ballot_sync(FULL_MASK, valid);
    if (valid) {
        unsigned peers = __match_any_sync(vmask, b);
        unsigned cnt = __reduce_add_sync(peers, 1u);
        if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(&hist[b], cnt);
    }
}
// warp-aggregated add returning this lane's rank (all lanes must call)
__device__ __forceinline__ uint32_t hist_rank_warp(uint32_t* hist, uint32_t b, bool valid) {
    unsigned vmask = __ballot_sync(FULL_MASK, valid);
    uint32_t rank = 0;
    unsigned peers = 0;
    int leader = 0;
    uint32_t old = 0;
    const int lane = threadIdx.x & 31;
    if (valid) {
        peers = __match_any_sync(vmask, b);
        leader = __ffs(peers) - 1;
        if (lane == leader) old = atomicAdd(&hist[b], (uint32_t)__popc(peers));
    }
    old = __shfl_sync(FULL_MASK, old, leader);
    if (valid) rank = old + __popc(peers & ((1u << lane) - 1u));
    return rank;
}

__device__ __forceinline__ uint32_t find_seg(const uint64_t* prefix, uint32_t nsegs, uint64_t tile) {
    uint32_t lo = 0, hi = nsegs;  // last s with prefix[s] <= tile
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
    uint64_t single[2];
    __device__ __forceinline__ void init(const void* base, uint64_t l, uint64_t h) {
        lo = l; hi = h;
        uint64_t par = (((uintptr_t)base) >> 3) & 1;
        a0 = lo + ((lo + par) & 1);
        if (a0 > hi) a0 = hi;
        npairs = (uint32_t)((hi - a0) / 2);
        nsingle = 0;
        if (a0 > lo) single[nsingle++] = lo;
        uint64_t t = a0 + 2ull * npairs;
        if (t < hi) single[nsingle++] = t;
    }
};

constexpr int kPairsPerThread = kTileKeys / (2 * kPartNT);  // 4

// ------------------------------------------------------- classify + hist
template <bool IN_F64, uint32_t KIND>
__device__ __forceinline__ void hist_tile(const Classifier& C, const void* src, const TileGeom& g,
                                          uint32_t* hist, Ctrl* ctrl) {
    const ulonglong2* sp = (const ulonglong2*)((const uint64_t*)src + g.a0);
    ulonglong2 v[kPairsPerThread];
#pragma unroll
    for (int j = 0; j < kPairsPerThread; ++j) {
        uint32_t p = threadIdx.x + j * kPartNT;
        if (p < g.npairs) v[j] = __ldcs(sp + p);
    }
#pragma unroll
    for (int j = 0; j < kPairsPerThread; ++j) {
        uint32_t p = threadIdx.x + j * kPartNT;
        bool ok = p < g.npairs;
        uint64_t k0 = v[j].x, k1 = v[j].y;
        if (IN_F64) {
            if (ok) {
                double d0 = __longlong_as_double((long long)k0), d1 = __longlong_as_double((long long)k1);
                if (isnan(d0)) atomicMin(&ctrl->nan_index, (unsigned long long)(g.a0 + 2 * p));
                if (isnan(d1)) atomicMin(&ctrl->nan_index, (unsigned long long)(g.a0 + 2 * p + 1));
            }
            k0 = encode(__longlong_as_double((long long)k0));
            k1 = encode(__longlong_as_double((long long)k1));
        }
        uint32_t b0 = ok ? C.classify<KIND>(k0) : 0;
        uint32_t b1 = ok ? C.classify<KIND>(k1) : 0;
        hist_add_warp(hist, b0 & 0x7fffffffu, ok);
        hist_add_warp(hist, b1 & 0x7fffffffu, ok);
    }
    if (threadIdx.x < g.nsingle) {
        uint64_t i = g.single[threadIdx.x];
        uint64_t k = ((const uint64_t*)src)[i];
        if (IN_F64) {
            double d = __longlong_as_double((long long)k);
            if (isnan(d)) atomicMin(&ctrl->nan_index, (unsigned long long)i);
            k = encode(d);
        }
        atomicAdd(&hist[C.classify<KIND>(k) & 0x7fffffffu], 1u);
    }
}

template <bool IN_F64>
__global__ void __launch_bounds__(kPartNT, 2) k_classify_hist(LevelParams p, uint32_t max_payload) {
    extern __shared__ uint4 smem_u4[];
    uint8_t* smem = (uint8_t*)smem_u4;
    uint8_t* msm = smem;
    uint32_t* hist = (uint32_t*)(smem + sizeof(ModelHdr) + max_payload);
    if (!IN_F64 && p.ctrl->nan_index != ~0ull) return;
    uint64_t per = (p.ntiles + gridDim.x - 1) / gridDim.x;
    uint64_t t0 = (uint64_t)blockIdx.x * per;
    uint64_t t1 = min(t0 + per, p.ntiles);
    int64_t cur = -1;
    Classifier C;
    uint32_t nb = 0;
    uint64_t boff = 0;
    for (uint64_t tile = t0; tile < t1; ++tile) {
        uint32_t s = find_seg(p.tile_prefix, p.nsegs, tile);
        if ((int64_t)s != cur) {
            if (cur >= 0) {
                __syncthreads();
                for (uint32_t b = threadIdx.x; b < nb; b += kPartNT)
                    if (hist[b]) atomicAdd(&p.buckets[boff + b], (unsigned long long)hist[b]);
                __syncthreads();
            }
            const SegDesc sd = p.segs[s];
            load_model_smem(p.models + sd.model_off, msm);
            C.init(msm);
            nb = C.nb;
            boff = sd.bucket_off;
            for (uint32_t b = threadIdx.x; b < nb; b += kPartNT) hist[b] = 0;
            __syncthreads();
            cur = s;
        }
        const SegDesc& sd = p.segs[s];
        uint64_t lo = sd.begin + (tile - p.tile_prefix[s]) * (uint64_t)kTileKeys;
        uint64_t hi = min(lo + kTileKeys, sd.begin + sd.n);
        TileGeom g;
        g.init(p.src, lo, hi);
        switch (C.kind) {
        case kLearned: hist_tile<IN_F64, kLearned>(C, p.src, g, hist, p.ctrl); break;
        case kTree: hist_tile<IN_F64, kTree>(C, p.src, g, hist, p.ctrl); break;
        case kRadix: hist_tile<IN_F64, kRadix>(C, p.src, g, hist, p.ctrl); break;
        default: hist_tile<IN_F64, kFill>(C, p.src, g, hist, p.ctrl); break;
        }
    }
    if (cur >= 0) {
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < nb; b += kPartNT)
            if (hist[b]) atomicAdd(&p.buckets[boff + b], (unsigned long long)hist[b]);
    }
}

// ---------------------------------------------------------- scan children
constexpr int kScanNT = 512;
__global__ void __launch_bounds__(kScanNT) k_scan_children(LevelParams p) {
    __shared__ uint64_t wsum[kScanNT / 32 + 1];
    __shared__ uint8_t iseq[kMaxNB];
    __shared__ uint64_t eqval[kMaxNB];
    extern __shared__ uint64_t cnt[];
    if (p.ctrl->nan_index != ~0ull) return;
    const SegDesc sd = p.segs[blockIdx.x];
    const uint8_t* mg = p.models + sd.model_off;
    const ModelHdr h = *(const ModelHdr*)mg;
    const uint32_t nb = h.nbuckets;
    for (uint32_t b = threadIdx.x; b < nb; b += kScanNT) {
        cnt[b] = p.buckets[sd.bucket_off + b];
        iseq[b] = 0;
    }
    __syncthreads();
    if (h.kind == kTree) {
        MView m = model_view(mg);
        for (uint32_t i = threadIdx.x; i < h.nsplit; i += kScanNT) {
            if (m.eqo[i + 1] - m.eqo[i] > 1) {
                iseq[m.eqo[i] + 1] = 1;
                eqval[m.eqo[i] + 1] = m.spl[i];
            }
        }
    } else if (h.kind == kFill && threadIdx.x == 0) {
        iseq[0] = 1;
        eqval[0] = h.radix_min;
    }
    __syncthreads();
    // keep counts: scan a copy held in registers per thread chunk
    block_exclusive_scan_u64<kScanNT>(cnt, nb, wsum);
    for (uint32_t b = threadIdx.x; b < nb; b += kScanNT) {
        uint64_t start = cnt[b];
        uint64_t end = (b + 1 < nb) ? cnt[b + 1] : sd.n;
        uint64_t len = end - start;
        uint64_t begin = sd.begin + start;
        p.buckets[sd.bucket_off + b] = begin;  // write cursor
        if (len == 0) continue;
        if (iseq[b]) {
            unsigned e = atomicAdd(&p.ctrl->n_fill, 1u);
            if (e < p.list_cap) p.fill[e] = FillItem{begin, len, eqval[b], 0};
            else atomicOr(&p.ctrl->err, 1u);
            atomicAdd(&p.ctrl->keys_fill, (unsigned long long)len);
        } else if (len <= p.base_cap[2]) {
            int c = len <= p.base_cap[0] ? 0 : (len <= p.base_cap[1] ? 1 : 2);
            unsigned e = atomicAdd(&p.ctrl->n_base[c], 1u);
            if (e < p.list_cap) p.base[c][e] = BaseItem{begin, len};
            else atomicOr(&p.ctrl->err, 2u);
            atomicAdd(&p.ctrl->keys_base, (unsigned long long)len);
        } else {
            unsigned e = atomicAdd(&p.ctrl->n_rec, 1u);
            uint32_t depth = sd.depth + 1;
            uint32_t flags = (len == sd.n || depth > p.depth_cap) ? kSegForceRadix : 0u;
            if (e < p.list_cap) p.rec[e] = SegOut{begin, len, depth, flags, 0};
            else atomicOr(&p.ctrl->err, 4u);
            atomicAdd(&p.ctrl->keys_rec, (unsigned long long)len);
        }
    }
}

// ---------------------------------------------------------------- scatter
template <bool IN_F64, bool MAPPED, uint32_t KIND>
__device__ __forceinline__ void scatter_tile(const Classifier& C, const LevelParams& p, const TileGeom& g,
                                             uint32_t nbo, uint64_t boff, uint32_t* cnt, uint32_t* lstart,
                                             unsigned long long* gpos, uint64_t* skeys, uint16_t* sbid,
                                             uint32_t* wsum, const uint32_t* map) {
    for (uint32_t b = threadIdx.x; b < nbo; b += kPartNT) cnt[b] = 0;
    __syncthreads();
    const ulonglong2* sp = (const ulonglong2*)((const uint64_t*)p.src + g.a0);
    ulonglong2 v[kPairsPerThread];
    uint32_t code[2 * kPairsPerThread];  // bucket << 16 | rank, 0xffffffff = skip
#pragma unroll
    for (int j = 0; j < kPairsPerThread; ++j) {
        uint32_t q = threadIdx.x + j * kPartNT;
        if (q < g.npairs) v[j] = __ldcs(sp + q);
    }
#pragma unroll
    for (int j = 0; j < kPairsPerThread; ++j) {
        uint32_t q = threadIdx.x + j * kPartNT;
        bool ok = q < g.npairs;
        if (IN_F64) {
            v[j].x = encode(__longlong_as_double((long long)v[j].x));
            v[j].y = encode(__longlong_as_double((long long)v[j].y));
        }
        uint32_t c0 = ok ? C.classify<KIND>(v[j].x) : (1u << 31);
        uint32_t c1 = ok ? C.classify<KIND>(v[j].y) : (1u << 31);
        bool ok0 = !(c0 >> 31), ok1 = !(c1 >> 31);
        uint32_t b0 = c0 & 0x7fffffffu, b1 = c1 & 0x7fffffffu;
        if (MAPPED) { if (ok0) b0 = map[b0]; if (ok1) b1 = map[b1]; }
        uint32_t r0 = hist_rank_warp(cnt, b0, ok0);
        uint32_t r1 = hist_rank_warp(cnt, b1, ok1);
        code[2 * j] = ok0 ? (b0 << 16 | r0) : 0xffffffffu;
        code[2 * j + 1] = ok1 ? (b1 << 16 | r1) : 0xffffffffu;
    }
    uint64_t sk[2] = {0, 0};
    uint32_t sc[2] = {0xffffffffu, 0xffffffffu};
    if (threadIdx.x < g.nsingle) {
        uint64_t k = load_key(p.src, g.single[threadIdx.x], IN_F64);
        uint32_t c = C.classify<KIND>(k);
        if (!(c >> 31)) {
            uint32_t b = c & 0x7fffffffu;
            if (MAPPED) b = map[b];
            uint32_t r = atomicAdd(&cnt[b], 1u);
            sk[0] = k;
            sc[0] = b << 16 | r;
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nbo; b += kPartNT) lstart[b] = cnt[b];
    __syncthreads();
    uint32_t total = block_exclusive_scan_u32<kPartNT>(lstart, nbo, wsum);
    for (uint32_t b = threadIdx.x; b < nbo; b += kPartNT)
        if (cnt[b]) gpos[b] = atomicAdd(&p.buckets[boff + b], (unsigned long long)cnt[b]);
#pragma unroll
    for (int j = 0; j < kPairsPerThread; ++j) {
        uint32_t c0 = code[2 * j], c1 = code[2 * j + 1];
        if (c0 != 0xffffffffu) {
            uint32_t pos = lstart[c0 >> 16] + (c0 & 0xffffu);
            skeys[pos] = v[j].x;
            sbid[pos] = (uint16_t)(c0 >> 16);
        }
        if (c1 != 0xffffffffu) {
            uint32_t pos = lstart[c1 >> 16] + (c1 & 0xffffu);
            skeys[pos] = v[j].y;
            sbid[pos] = (uint16_t)(c1 >> 16);
        }
    }
    if (sc[0] != 0xffffffffu) {
        uint32_t pos = lstart[sc[0] >> 16] + (sc[0] & 0xffffu);
        skeys[pos] = sk[0];
        sbid[pos] = (uint16_t)(sc[0] >> 16);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < total; j += kPartNT) {
        uint32_t b = sbid[j];
        p.dst[gpos[b] + (j - lstart[b])] = skeys[j];
    }
    __syncthreads();
}

template <bool IN_F64, bool MAPPED>
__global__ void __launch_bounds__(kPartNT, 2) k_scatter(LevelParams p, uint32_t max_payload, uint32_t max_nb,
                                                    const uint32_t* map, uint32_t nmapped) {
    extern __shared__ uint4 smem_u4[];
    uint8_t* smem = (uint8_t*)smem_u4;
    uint8_t* msm = smem;
    uint8_t* q = smem + sizeof(ModelHdr) + max_payload;
    uint32_t nbo_max = MAPPED ? nmapped : max_nb;
    unsigned long long* gpos = (unsigned long long*)q; q += 8 * (size_t)nbo_max;
    uint64_t* skeys = (uint64_t*)q; q += 8 * (size_t)kTileKeys;
    uint32_t* cnt = (uint32_t*)q; q += 4 * (size_t)nbo_max;
    uint32_t* lstart = (uint32_t*)q; q += 4 * (size_t)(nbo_max + 1);
    uint32_t* wsum = (uint32_t*)q; q += 4 * (kPartNT / 32 + 1);
    uint16_t* sbid = (uint16_t*)q;
    if (p.ctrl->nan_index != ~0ull) return;
    uint64_t per = (p.ntiles + gridDim.x - 1) / gridDim.x;
    uint64_t t0 = (uint64_t)blockIdx.x * per;
    uint64_t t1 = min(t0 + per, p.ntiles);
    int64_t cur = -1;
    Classifier C;
    uint64_t boff = 0;
    for (uint64_t tile = t0; tile < t1; ++tile) {
        uint32_t s = find_seg(p.tile_prefix, p.nsegs, tile);
        if ((int64_t)s != cur) {
            __syncthreads();
            const SegDesc sd = p.segs[s];
            load_model_smem(p.models + sd.model_off, msm);
            C.init(msm);
            boff = sd.bucket_off;
            cur = s;
        }
        const SegDesc& sd = p.segs[s];
        uint64_t lo = sd.begin + (tile - p.tile_prefix[s]) * (uint64_t)kTileKeys;
        uint64_t hi = min(lo + kTileKeys, sd.begin + sd.n);
        TileGeom g;
        g.init(p.src, lo, hi);
        uint32_t nbo = MAPPED ? nmapped : C.nb;
        switch (C.kind) {
        case kLearned: scatter_tile<IN_F64, MAPPED, kLearned>(C, p, g, nbo, boff, cnt, lstart, gpos, skeys, sbid, wsum, map); break;
        case kTree: scatter_tile<IN_F64, MAPPED, kTree>(C, p, g, nbo, boff, cnt, lstart, gpos, skeys, sbid, wsum, map); break;
        case kRadix: scatter_tile<IN_F64, MAPPED, kRadix>(C, p, g, nbo, boff, cnt, lstart, gpos, skeys, sbid, wsum, map); break;
        default: break;  // kFill: nothing moves
        }
    }
}

// -------------------------------------------------------------- base case
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
    uint32_t ni = min(*count, list_cap);
    for (uint32_t e = blockIdx.x; e < ni; e += gridDim.x) {
        const BaseItem it = items[e];
        const uint32_t n = (uint32_t)it.n;
        if (n == 1) {
            if (threadIdx.x == 0) {
                uint64_t k = src[it.begin];
                if (OUT_F64) ((double*)out)[it.begin] = decode(k);
                else ((uint64_t*)out)[it.begin] = k;
            }
            continue;
        }
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
    uint32_t ni = min(*count, list_cap);
    uint64_t chunk0 = 0;
    for (uint32_t e = 0; e < ni; ++e) {
        const FillItem it = items[e];
        uint64_t nch = (it.n + kFillChunk - 1) / kFillChunk;
        uint64_t first = (blockIdx.x + gridDim.x - (chunk0 % gridDim.x)) % gridDim.x;
        uint64_t v = OUT_F64 ? (uint64_t)__double_as_longlong(decode(it.value)) : it.value;
        for (uint64_t c = first; c < nch; c += gridDim.x) {
            uint64_t lo = it.begin + c * kFillChunk;
            uint64_t hi = min(lo + kFillChunk, it.begin + it.n);
            for (uint64_t i = lo + threadIdx.x; i < hi; i += 256) __stcs((unsigned long long*)out + i, v);
        }
        chunk0 += nch;
    }
}

// ------------------------------------------------------- model building
// Fold step of the reference's running max (std::max(lo[m], lo[m-1]),
// models.cpp:110): keep the new element unless it is strictly smaller.
struct StepMax { __device__ double operator()(double acc, double e) const { return (e < acc) ? acc : e; } };
// std::min(hi[m], hi[m+1]) folded right to left (models.cpp:111)
struct StepMin { __device__ double operator()(double acc, double e) const { return (acc < e) ? acc : e; } };

// Inclusive sequential-fold scan of a[0,n) in processing order (reverse =
// right to left). Each step is `acc = op(acc, e)`; chunked per thread, with
// chunk carries combined by the same op (exact for these fold rules).
template <int NT, class Op>
__device__ void block_fold_scan(double* a, uint32_t n, bool reverse, double* wtmp, Op op) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t per = (n + NT - 1) / NT;
    const uint32_t lo = threadIdx.x * per, hi = min(lo + per, n);
    auto at = [&](uint32_t i) -> double& { return reverse ? a[n - 1 - i] : a[i]; };
    bool have = lo < hi;
    double acc = 0.0;
    if (have) {
        acc = at(lo);
        for (uint32_t i = lo + 1; i < hi; ++i) acc = op(acc, at(i));
    }
    // exclusive carry across threads in order
    double inc = acc;
    bool hinc = have;
    for (int o = 1; o < 32; o <<= 1) {
        double w = __shfl_up_sync(FULL_MASK, inc, o);
        bool hw = __shfl_up_sync(FULL_MASK, (int)hinc, o);
        if (lane >= o && hw) { inc = hinc ? op(w, inc) : w; hinc = true; }
    }
    __syncthreads();
    if (lane == 31) { wtmp[2 * warp] = inc; wtmp[2 * warp + 1] = hinc ? 1.0 : 0.0; }
    __syncthreads();
    if (warp == 0) {
        double x = lane < NT / 32 ? wtmp[2 * lane] : 0.0;
        bool hx = lane < NT / 32 ? wtmp[2 * lane + 1] != 0.0 : false;
        double ix = x;
        bool hix = hx;
        for (int o = 1; o < 32; o <<= 1) {
            double w = __shfl_up_sync(FULL_MASK, ix, o);
            bool hw = __shfl_up_sync(FULL_MASK, (int)hix, o);
            if (lane >= o && hw) { ix = hix ? op(w, ix) : w; hix = true; }
        }
        // exclusive for warp `lane`: inclusive of lane-1
        double ex = __shfl_up_sync(FULL_MASK, ix, 1);
        bool hex = __shfl_up_sync(FULL_MASK, (int)hix, 1);
        if (lane == 0) hex = false;
        __syncwarp();
        if (lane < NT / 32) { wtmp[2 * lane] = ex; wtmp[2 * lane + 1] = hex ? 1.0 : 0.0; }
    }
    __syncthreads();
    // carry for this thread = warp carry combined with lanes before it
    double wc = wtmp[2 * warp];
    bool hwc = wtmp[2 * warp + 1] != 0.0;
    double lex = __shfl_up_sync(FULL_MASK, inc, 1);
    bool hlex = __shfl_up_sync(FULL_MASK, (int)hinc, 1);
    if (lane == 0) hlex = false;
    double carry = 0.0;
    bool hc = false;
    if (hwc) { carry = wc; hc = true; }
    if (hlex) { carry = hc ? op(carry, lex) : lex; hc = true; }
    if (have) {
        double x = hc ? op(carry, at(lo)) : at(lo);
        at(lo) = x;
        for (uint32_t i = lo + 1; i < hi; ++i) { x = op(x, at(i)); at(i) = x; }
    }
    __syncthreads();
}

__device__ __forceinline__ double dmax_ref(double a, double b) { return (a < b) ? b : a; }  // std::max
__device__ __forceinline__ double dmin_ref(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double dclamp01(double v) { return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v); }

// Sequential fit_line (models.cpp:14-35) over [first,last) -- bit-exact.
struct Fit { double slope, intercept; };
template <class XN>
__device__ Fit fit_seq(XN xn, uint32_t first, uint32_t last, double inv_n_total, double n_total) {
    uint32_t n = last - first;
    if (n == 0) return {0.0, 0.0};
    double sx = 0.0, sy = 0.0;
    for (uint32_t i = first; i < last; ++i) {
        sx = __dadd_rn(sx, xn(i));
        sy = __dadd_rn(sy, __ddiv_rn((double)i, n_total));
    }
    double mx = __ddiv_rn(sx, (double)n), my = __ddiv_rn(sy, (double)n);
    double sxx = 0.0, sxy = 0.0;
    for (uint32_t i = first; i < last; ++i) {
        double dx = __dsub_rn(xn(i), mx);
        sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
        sxy = __dadd_rn(sxy, __dmul_rn(dx, __dsub_rn(__ddiv_rn((double)i, n_total), my)));
    }
    if (!(sxx > 0.0)) return {0.0, my};
    double slope = __ddiv_rn(sxy, sxx);
    if (slope < 0.0) return {0.0, my};
    return {slope, __dsub_rn(my, __dmul_rn(slope, mx))};
}

// Warp-cooperative fit (deterministic lane-chunk order; not the reference's
// sequential order: within a few ulps of it).
template <class XN>
__device__ Fit fit_warp(XN xn, uint32_t first, uint32_t last, double n_total) {
    const int lane = threadIdx.x & 31;
    uint32_t n = last - first;
    uint32_t per = (n + 31) / 32;
    uint32_t lo = first + min(n, lane * per), hi = first + min(n, (lane + 1) * per);
    double sx = 0.0, sy = 0.0;
    for (uint32_t i = lo; i < hi; ++i) {
        sx = __dadd_rn(sx, xn(i));
        sy = __dadd_rn(sy, __ddiv_rn((double)i, n_total));
    }
    for (int o = 1; o < 32; o <<= 1) {  // fixed-order pairwise tree
        double a = __shfl_down_sync(FULL_MASK, sx, o), b = __shfl_down_sync(FULL_MASK, sy, o);
        if ((lane & (2 * o - 1)) == 0) { sx = __dadd_rn(sx, a); sy = __dadd_rn(sy, b); }
    }
    sx = __shfl_sync(FULL_MASK, sx, 0);
    sy = __shfl_sync(FULL_MASK, sy, 0);
    double mx = __ddiv_rn(sx, (double)n), my = __ddiv_rn(sy, (double)n);
    double sxx = 0.0, sxy = 0.0;
    for (uint32_t i = lo; i < hi; ++i) {
        double dx = __dsub_rn(xn(i), mx);
        sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
        sxy = __dadd_rn(sxy, __dmul_rn(dx, __dsub_rn(__ddiv_rn((double)i, n_total), my)));
    }
    for (int o = 1; o < 32; o <<= 1) {
        double a = __shfl_down_sync(FULL_MASK, sxx, o), b = __shfl_down_sync(FULL_MASK, sxy, o);
        if ((lane & (2 * o - 1)) == 0) { sxx = __dadd_rn(sxx, a); sxy = __dadd_rn(sxy, b); }
    }
    sxx = __shfl_sync(FULL_MASK, sxx, 0);
    sxy = __shfl_sync(FULL_MASK, sxy, 0);
    if (!(sxx > 0.0)) return {0.0, my};
    double slope = __ddiv_rn(sxy, sxx);
    if (slope < 0.0) return {0.0, my};
    return {slope, __dsub_rn(my, __dmul_rn(slope, mx))};
}

// Rmi::train + enforce_monotonic (models.cpp:39-131) by one CTA over a sorted
// sample s[0,n) (shared or global memory). Scratch (shared): first[B+1] u32,
// lo[B], hi[B] doubles, big-slice list. Output: header + entries (global).
constexpr int kSeqFitMax = 512;
template <int NT>
__device__ void train_rmi_block(const uint64_t* s, uint32_t n, uint32_t B, ModelHdr* hdr, RmiEntry* E,
                                uint32_t* first, double* lo, double* hi, uint32_t* biglist, double* red) {
    const double base = __ull2double_rn(s[0]);
    const double kmax = __ull2double_rn(s[n - 1]);
    const double scale = kmax > base ? __ddiv_rn(1.0, __dsub_rn(kmax, base)) : 0.0;
    const double nd = (double)n;
    auto xn = [&](uint32_t i) { return rmi_normalize(base, scale, s[i]); };
    // root fit_line over the whole sample: deterministic block reduction
    const uint32_t per = (n + NT - 1) / NT;
    const uint32_t lo0 = min(n, threadIdx.x * per), hi0 = min(n, lo0 + per);
    double sx = 0.0, sy = 0.0;
    for (uint32_t i = lo0; i < hi0; ++i) {
        sx = __dadd_rn(sx, xn(i));
        sy = __dadd_rn(sy, __ddiv_rn((double)i, nd));
    }
    sx = block_sum_f64<NT>(sx, red);
    sy = block_sum_f64<NT>(sy, red);
    const double mx = __ddiv_rn(sx, nd), my = __ddiv_rn(sy, nd);
    double sxx = 0.0, sxy = 0.0;
    for (uint32_t i = lo0; i < hi0; ++i) {
        double dx = __dsub_rn(xn(i), mx);
        sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
        sxy = __dadd_rn(sxy, __dmul_rn(dx, __dsub_rn(__ddiv_rn((double)i, nd), my)));
    }
    sxx = block_sum_f64<NT>(sxx, red);
    sxy = block_sum_f64<NT>(sxy, red);
    double rs, ri;
    if (!(sxx > 0.0)) { rs = 0.0; ri = my; }
    else {
        double sl = __ddiv_rn(sxy, sxx);
        if (sl < 0.0) { rs = 0.0; ri = my; }
        else { rs = sl; ri = __dsub_rn(my, __dmul_rn(sl, mx)); }
    }
    // fit_line never returns a negative slope, so enforce_monotonic's
    // root/submodel negative-slope repairs (models.cpp:83-86,99-100) are no-ops.
    // Slice boundaries: first[m] = min{i : route(xn(i)) >= m} (routes are
    // nondecreasing along the sorted sample).
    for (uint32_t m = threadIdx.x; m <= B; m += NT) {
        uint32_t a = 0, b = n;
        if (m == 0) b = 0;
        else if (m == B) a = n;
        while (a < b) {
            uint32_t mid = (a + b) >> 1;
            if (rmi_route(rs, ri, B, xn(mid)) >= m) b = mid; else a = mid + 1;
        }
        first[m] = a;
    }
    __shared__ uint32_t nbig;
    if (threadIdx.x == 0) nbig = 0;
    __syncthreads();
    for (uint32_t m = threadIdx.x; m < B; m += NT) {
        uint32_t f = first[m], l = first[m + 1];
        if (l - f > (uint32_t)kSeqFitMax) {
            biglist[atomicAdd(&nbig, 1u)] = m;
            continue;
        }
        Fit ft = fit_seq(xn, f, l, 0.0, nd);
        E[m].slope = ft.slope;
        E[m].intercept = ft.intercept;
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x >> 5; q < nbig; q += NT / 32) {
        uint32_t m = biglist[q];
        Fit ft = fit_warp(xn, first[m], first[m + 1], nd);
        if ((threadIdx.x & 31) == 0) {
            E[m].slope = ft.slope;
            E[m].intercept = ft.intercept;
        }
    }
    __syncthreads();
    // enforce_monotonic (models.cpp:101-126)
    for (uint32_t m = threadIdx.x; m < B; m += NT) {
        uint32_t f = first[m], l = first[m + 1];
        if (l > f) {
            double sl = E[m].slope, ic = E[m].intercept;
            lo[m] = __dadd_rn(__dmul_rn(sl, xn(f)), ic);
            hi[m] = __dadd_rn(__dmul_rn(sl, xn(l - 1)), ic);
        } else {
            lo[m] = -INFINITY;
            hi[m] = INFINITY;
        }
    }
    __syncthreads();
    block_fold_scan<NT>(lo, B, false, red, StepMax());
    block_fold_scan<NT>(hi, B, true, red, StepMin());
    double* hi2 = lo + B;  // lo/hi arrays are adjacent? use registers instead
    (void)hi2;
    for (uint32_t m = threadIdx.x; m < B; m += NT) {
        double h = hi[m];
        if (m + 1 < B) h = dmin_ref(h, lo[m + 1]);
        h = dmax_ref(h, lo[m]);
        double l = dclamp01(lo[m]);
        h = dclamp01(h);
        if (m == 0) l = 0.0;
        if (m == B - 1) h = 1.0;
        if (first[m + 1] == first[m]) {
            E[m].slope = 0.0;
            E[m].intercept = __dmul_rn(0.5, __dadd_rn(l, h));
        }
        E[m].lo = l;
        E[m].hi = h;
    }
    if (threadIdx.x == 0) {
        hdr->root_slope = rs;
        hdr->root_icpt = ri;
        hdr->key_base = base;
        hdr->key_scale = scale;
        hdr->B = B;
    }
    __syncthreads();
}

// SplitterTree::build (models.cpp:133-185) by one CTA from a sorted sample in
// shared memory. Scratch: u32[2k].
template <int NT>
__device__ void tree_build_block(const uint64_t* s, uint32_t n, uint32_t k, bool eq_mode, ModelHdr* hdr,
                                 uint8_t* payload, uint32_t* scratch, uint32_t* wsum, uint64_t* spl_tmp) {
    uint32_t* keep = scratch;      // k entries
    uint32_t* eqo = scratch + k;   // k entries (+1)
    for (uint32_t i = threadIdx.x; i + 1 < k; i += NT) {
        uint64_t q = (uint64_t)(i + 1) * n / k;
        uint32_t pos = (uint32_t)((q > 1 ? q : 1) - 1);
        uint64_t v = s[pos];
        bool kp = true;
        if (i > 0) {
            uint64_t qp = (uint64_t)i * n / k;
            uint32_t pp = (uint32_t)((qp > 1 ? qp : 1) - 1);
            kp = v > s[pp];
        }
        keep[i] = kp ? 1u : 0u;
    }
    __syncthreads();
    uint32_t m = block_exclusive_scan_u32<NT>(keep, k - 1, wsum);
    for (uint32_t i = threadIdx.x; i + 1 < k; i += NT) {
        uint32_t nxt = (i + 2 < k) ? keep[i + 1] : m;
        if (nxt != keep[i]) {  // kept
            uint64_t q = (uint64_t)(i + 1) * n / k;
            uint32_t pos = (uint32_t)((q > 1 ? q : 1) - 1);
            spl_tmp[keep[i]] = s[pos];
        }
    }
    __syncthreads();
    if (m == 0) {  // defensive (k >= 2 always keeps candidate 0)
        if (threadIdx.x == 0) spl_tmp[0] = s[0];
        m = 1;
        __syncthreads();
    }
    for (uint32_t j = threadIdx.x; j < m; j += NT) {
        uint64_t v = spl_tmp[j];
        uint32_t a = 0, b = n;  // lower_bound
        while (a < b) { uint32_t mid = (a + b) >> 1; if (s[mid] < v) a = mid + 1; else b = mid; }
        uint32_t f = a;
        b = n;  // upper_bound
        while (a < b) { uint32_t mid = (a + b) >> 1; if (v < s[mid]) b = mid; else a = mid + 1; }
        uint64_t count = a - f;
        bool heavy = eq_mode && count * (uint64_t)k > (uint64_t)n;
        eqo[j] = heavy ? 2u : 1u;
    }
    __syncthreads();
    uint32_t total = block_exclusive_scan_u32<NT>(eqo, m, wsum);
    if (threadIdx.x == 0) eqo[m] = total;
    __syncthreads();
    uint32_t levels = 1;
    while ((1u << levels) < m + 1) ++levels;
    uint32_t leaf = 1u << levels;
    uint64_t* tree = (uint64_t*)payload;
    uint64_t* spl = tree + leaf;
    uint32_t* eq_out = (uint32_t*)(spl + m);
    for (uint32_t j = threadIdx.x; j < leaf; j += NT) {
        if (j == 0) { tree[0] = 0; continue; }
        uint32_t d = 31 - __clz(j);
        uint32_t pidx = j - (1u << d);
        uint32_t io = ((2 * pidx + 1) << (levels - 1 - d)) - 1;
        tree[j] = io < m ? spl_tmp[io] : ~0ull;
    }
    for (uint32_t j = threadIdx.x; j < m; j += NT) spl[j] = spl_tmp[j];
    for (uint32_t j = threadIdx.x; j <= m; j += NT) eq_out[j] = eqo[j];
    if (threadIdx.x == 0) {
        hdr->kind = kTree;
        hdr->levels = levels;
        hdr->leaf_origin = leaf;
        hdr->nsplit = m;
        hdr->nbuckets = total + 1;
    }
    __syncthreads();
}

constexpr int kModelNT = 512;
using ModelSort = BlockSort<kModelNT, 32, 8192>;
struct ModelSmem {
    uint64_t a[16384];
    union {
        typename ModelSort::Smem sort;
        struct {
            uint32_t first[LSORT_MAX_RMI_DEV + 1];
            double lo[LSORT_MAX_RMI_DEV];
            double hi[LSORT_MAX_RMI_DEV];
            uint32_t big[LSORT_MAX_RMI_DEV];
            double red[2 * (kModelNT / 32)];
        } rmi;
        struct {
            uint32_t scratch[2 * LSORT_MAX_TREE_DEV + 2];
            uint32_t wsum[kModelNT / 32 + 1];
            uint64_t spl[LSORT_MAX_TREE_DEV];
        } tree;
    } u;
    uint64_t red64[kModelNT / 32];
    uint32_t distinct;
};

// Radix/fill fallback model: min/max of the whole segment (one CTA).
__device__ void build_radix_model(const SegDesc& sd, const void* src, bool f64, ModelHdr* h, uint64_t* red) {
    uint64_t mn = ~0ull, mx = 0;
    for (uint64_t i = threadIdx.x; i < sd.n; i += kModelNT) {
        uint64_t k = load_key(src, sd.begin + i, f64);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    mn = block_reduce_min<kModelNT>(mn, red);
    mx = block_reduce_max<kModelNT>(mx, red);
    if (threadIdx.x == 0) {
        if (mn == mx) {
            h->kind = kFill;
            h->nbuckets = 1;
        } else {
            uint32_t bits = bitlen64(mx - mn);
            h->kind = kRadix;
            h->shift = bits > kRadixBits ? bits - kRadixBits : 0;
            h->nbuckets = (uint32_t)((mx - mn) >> h->shift) + 1;
        }
        h->radix_min = mn;
    }
    __syncthreads();
}

// Alg. 5 build_partition_model for one segment.
template <bool IN_F64>
__device__ void build_model_cta(const SegDesc& sd, const void* src, uint8_t* models, const DevCfg& cfg,
                                ModelSmem& S, bool first_only) {
    ModelHdr* h = (ModelHdr*)(models + sd.model_off);
    uint8_t* payload = models + sd.model_off + sizeof(ModelHdr);
    if (sd.flags & kSegForceRadix) {
        build_radix_model(sd, src, IN_F64, h, S.red64);
        return;
    }
    const uint64_t n = sd.n;
    const uint64_t seed = seg_seed(cfg.seed, sd.begin, sd.depth);
    const uint32_t s1 = (uint32_t)first_sample_size(cfg, n);
    uint64_t k[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        uint32_t idx = threadIdx.x + i * kModelNT;
        if (idx < s1) k[i] = load_key(src, sd.begin + sample_index(seed, idx, n), IN_F64);
    }
    ModelSort::sort_regs(k, S.a, s1, S.u.sort);
    __syncthreads();
    uint64_t d = 0;
    for (uint32_t i = threadIdx.x + 1; i < s1; i += kModelNT) d += S.a[i] != S.a[i - 1];
    d = block_reduce_sum_u64<kModelNT>(d, S.red64);
    const uint64_t distinct = 1 + d;
    const double dup = __dsub_rn(1.0, __ddiv_rn((double)distinct, (double)s1));  // models.cpp:187-193
    const bool learned = n >= cfg.min_rmi_input && dup <= cfg.max_dup;
    if (threadIdx.x == 0) {
        h->dup = dup;
        h->s1 = s1;
        h->flags = 0;
        h->cdf_lo = 0.0;
        h->inv_span = 1.0;  // Learned::inv_span() with cdf [0,1] (models.hpp:134-137)
    }
    if (learned) {
        const uint32_t s2 = (uint32_t)rmi_sample_size(cfg, n);
        if (threadIdx.x == 0) {
            h->kind = kLearned;
            h->nbuckets = sd.rmi_b;
            h->B = sd.rmi_b;
            h->s2 = s2;
        }
        if (first_only) { __syncthreads(); return; }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            uint32_t idx = threadIdx.x + i * kModelNT;
            if (idx < s2) k[i] = load_key(src, sd.begin + sample_index(seed, s1 + idx, n), IN_F64);
        }
        __syncthreads();
        ModelSort::sort_regs(k, S.a, s2, S.u.sort);
        __syncthreads();
        train_rmi_block<kModelNT>(S.a, s2, sd.rmi_b, h, (RmiEntry*)payload, S.u.rmi.first, S.u.rmi.lo,
                                  S.u.rmi.hi, S.u.rmi.big, S.u.rmi.red);
    } else {
        if (threadIdx.x == 0) h->s2 = 0;
        tree_build_block<kModelNT>(S.a, s1, sd.tree_k, true, h, payload, S.u.tree.scratch, S.u.tree.wsum,
                                   S.u.tree.spl);
    }
}

template <bool IN_F64>
__global__ void __launch_bounds__(kModelNT) k_build_models(const SegDesc* segs, const uint32_t* idx, const void* src,
                                                          uint8_t* models, DevCfg cfg) {
    extern __shared__ uint4 smem_u4[];
    ModelSmem& S = *(ModelSmem*)smem_u4;
    const SegDesc sd = segs[idx[blockIdx.x]];
    build_model_cta<IN_F64>(sd, src, models, cfg, S, false);
}

template <bool IN_F64>
__global__ void __launch_bounds__(kModelNT) k_first_sample(const SegDesc* seg, const void* src, uint8_t* models,
                                                          DevCfg cfg) {
    extern __shared__ uint4 smem_u4[];
    ModelSmem& S = *(ModelSmem*)smem_u4;
    const SegDesc sd = *seg;
    build_model_cta<IN_F64>(sd, src, models, cfg, S, true);
}

template <bool IN_F64>
__global__ void k_gather(const SegDesc* seg, const void* src, uint64_t seed, uint64_t j0, uint64_t s,
                         uint64_t* out) {
    const SegDesc sd = *seg;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < s; j += (uint64_t)gridDim.x * blockDim.x)
        out[j] = load_key(src, sd.begin + sample_index(seed, j0 + j, sd.n), IN_F64);
}

constexpr int kTrainNT = 1024;
__global__ void __launch_bounds__(kTrainNT) k_train_rmi_global(const uint64_t* sample, uint64_t s, uint32_t B,
                                                              uint8_t* model, uint32_t nbuckets) {
    extern __shared__ uint4 smem_u4[];
    uint32_t* first = (uint32_t*)smem_u4;
    double* lo = (double*)(first + ((B + 1 + 1) & ~1u));
    double* hi = lo + B;
    uint32_t* big = (uint32_t*)(hi + B);
    double* red = (double*)(big + ((B + 1) & ~1u));
    ModelHdr* h = (ModelHdr*)model;
    train_rmi_block<kTrainNT>(sample, (uint32_t)s, B, h, (RmiEntry*)(model + sizeof(ModelHdr)), first, lo, hi, big,
                              red);
    if (threadIdx.x == 0) {
        h->kind = kLearned;
        h->nbuckets = nbuckets;
    }
}

// -------------------------------------------------------- unit / utility
template <bool IN_F64>
__global__ void __launch_bounds__(256) k_classify_ids(const uint8_t* model, const void* keys, uint64_t n, uint32_t* ids,
                                                     unsigned long long* hist) {
    extern __shared__ uint4 smem_u4[];
    uint8_t* msm = (uint8_t*)smem_u4;
    load_model_smem(model, msm);
    Classifier C;
    C.init(msm);
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        uint64_t k = load_key(keys, i, IN_F64);
        uint32_t b;
        switch (C.kind) {
        case kLearned: b = C.classify<kLearned>(k); break;
        case kTree: b = C.classify<kTree>(k); break;
        case kRadix: b = C.classify<kRadix>(k); break;
        default: b = C.classify<kFill>(k); break;
        }
        b &= 0x7fffffffu;
        if (ids) ids[i] = b;
        if (hist) atomicAdd(&hist[b], 1ull);
    }
}

__global__ void __launch_bounds__(kModelNT) k_tree_build(const uint64_t* sorted, uint32_t s, uint32_t budget, int eq_mode, uint8_t* model) {
    extern __shared__ uint4 smem_u4[];
    ModelSmem& S = *(ModelSmem*)smem_u4;
    for (uint32_t i = threadIdx.x; i < s; i += kModelNT) S.a[i] = sorted[i];
    __syncthreads();
    tree_build_block<kModelNT>(S.a, s, budget, eq_mode != 0, (ModelHdr*)model, model + sizeof(ModelHdr),
                               S.u.tree.scratch, S.u.tree.wsum, S.u.tree.spl);
}

__global__ void __launch_bounds__(kModelNT) k_block_sort(uint64_t* keys, uint32_t n) {
    extern __shared__ uint4 smem_u4[];
    ModelSmem& S = *(ModelSmem*)smem_u4;
    uint64_t k[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        uint32_t idx = threadIdx.x + i * kModelNT;
        if (idx < n) k[i] = keys[idx];
    }
    ModelSort::sort_regs(k, S.a, n, S.u.sort);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += kModelNT) keys[i] = S.a[i];
}

template <bool F64>
__global__ void __launch_bounds__(256) k_verify(const void* keys, uint64_t n, Ctrl* ctrl) {
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
    for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
        ((double*)keys)[i] = decode(keys[i]);
}

// ------------------------------------------------------------- launchers
static int g_num_sms = 148;

size_t model_smem_bytes() { return sizeof(ModelSmem); }

template <class F>
static void allow_smem(F* f, int optin) {
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, f) != cudaSuccess) { cudaGetLastError(); return; }
    int dyn = optin - (int)a.sharedSizeBytes;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn) != cudaSuccess) cudaGetLastError();
}

void kernels_init() {
    static bool done = false;
    if (done) return;
    done = true;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    int optin = 227 * 1024;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    allow_smem(k_classify_hist<true>, optin);
    allow_smem(k_classify_hist<false>, optin);
    allow_smem(k_scatter<true, false>, optin);
    allow_smem(k_scatter<false, false>, optin);
    allow_smem(k_scatter<true, true>, optin);
    allow_smem(k_scatter<false, true>, optin);
    allow_smem(k_scan_children, optin);
    allow_smem(k_build_models<true>, optin);
    allow_smem(k_build_models<false>, optin);
    allow_smem(k_first_sample<true>, optin);
    allow_smem(k_first_sample<false>, optin);
    allow_smem(k_train_rmi_global, optin);
    allow_smem(k_tree_build, optin);
    allow_smem(k_block_sort, optin);
    allow_smem(k_classify_ids<true>, optin);
    allow_smem(k_classify_ids<false>, optin);
    allow_smem(k_small_sort<true>, optin);
    allow_smem(k_small_sort<false>, optin);
    allow_smem(k_base<128, 8, 1024, true>, optin);
    allow_smem(k_base<128, 8, 1024, false>, optin);
    allow_smem(k_base<256, 16, 4096, true>, optin);
    allow_smem(k_base<256, 16, 4096, false>, optin);
    allow_smem(k_base<512, 32, 8192, true>, optin);
    allow_smem(k_base<512, 32, 8192, false>, optin);
}

int num_sms() { return g_num_sms; }

void launch_build_models(const SegDesc* segs, const uint32_t* idx, uint32_t count, const void* src, int in_f64,
                         uint8_t* models, const DevCfg& cfg, int, cudaStream_t st) {
    if (!count) return;
    size_t sm = sizeof(ModelSmem);
    if (in_f64) k_build_models<true><<<count, kModelNT, sm, st>>>(segs, idx, src, models, cfg);
    else k_build_models<false><<<count, kModelNT, sm, st>>>(segs, idx, src, models, cfg);
}

void launch_first_sample(const SegDesc* seg, const void* src, int in_f64, uint8_t* models, const DevCfg& cfg,
                         cudaStream_t st) {
    size_t sm = sizeof(ModelSmem);
    if (in_f64) k_first_sample<true><<<1, kModelNT, sm, st>>>(seg, src, models, cfg);
    else k_first_sample<false><<<1, kModelNT, sm, st>>>(seg, src, models, cfg);
}

void launch_gather(const SegDesc* seg, const void* src, int in_f64, uint64_t seed, uint64_t j0, uint64_t s,
                   uint64_t* out, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((s + 255) / 256, (uint64_t)g_num_sms * 8);
    if (in_f64) k_gather<true><<<grid, 256, 0, st>>>(seg, src, seed, j0, s, out);
    else k_gather<false><<<grid, 256, 0, st>>>(seg, src, seed, j0, s, out);
}

void launch_train_rmi_global(const uint64_t* sample, uint64_t s, uint32_t B, uint8_t* model, uint32_t nbuckets,
                             cudaStream_t st) {
    size_t sm = 4 * (size_t)((B + 2) & ~1u) + 16 * (size_t)B + 4 * (size_t)((B + 1) & ~1u) + 16 * (kTrainNT / 32) + 64;
    k_train_rmi_global<<<1, kTrainNT, sm, st>>>(sample, s, B, model, nbuckets);
}

static size_t part_smem_hist(int max_payload, int max_nb) {
    return sizeof(ModelHdr) + (size_t)max_payload + 4 * (size_t)max_nb;
}
static size_t part_smem_scatter(int max_payload, int nbo) {
    return sizeof(ModelHdr) + (size_t)max_payload + 8 * (size_t)nbo + 8 * (size_t)kTileKeys + 4 * (size_t)nbo +
           4 * (size_t)(nbo + 1) + 4 * (kPartNT / 32 + 1) + 2 * (size_t)kTileKeys + 16;
}

void launch_classify_hist(const LevelParams& p, int in_f64, int max_payload, int grid, cudaStream_t st) {
    if (!p.ntiles) return;
    uint32_t max_nb = 0;
    // the histogram region is sized for the widest segment (<= 2*LSORT_MAX_TREE or LSORT_MAX_RMI)
    max_nb = kMaxNB;
    size_t sm = part_smem_hist(max_payload, (int)max_nb);
    if (in_f64) k_classify_hist<true><<<grid, kPartNT, sm, st>>>(p, (uint32_t)max_payload);
    else k_classify_hist<false><<<grid, kPartNT, sm, st>>>(p, (uint32_t)max_payload);
}

void launch_scan_children(const LevelParams& p, cudaStream_t st) {
    if (!p.nsegs) return;
    size_t sm = 8 * kMaxNB;
    k_scan_children<<<p.nsegs, kScanNT, sm, st>>>(p);
}

void launch_scatter(const LevelParams& p, int in_f64, int max_payload, int max_nb, int grid, cudaStream_t st) {
    if (!p.ntiles) return;
    size_t sm = part_smem_scatter(max_payload, max_nb);
    if (in_f64) k_scatter<true, false><<<grid, kPartNT, sm, st>>>(p, (uint32_t)max_payload, (uint32_t)max_nb, nullptr, 0);
    else k_scatter<false, false><<<grid, kPartNT, sm, st>>>(p, (uint32_t)max_payload, (uint32_t)max_nb, nullptr, 0);
}

void launch_base_cases(const LevelParams& p, const uint64_t* src, void* out, uint64_t*, int out_f64, int grid_mult,
                       cudaStream_t st) {
    using S = BaseCfg<128, 8, 1024>;
    using M = BaseCfg<256, 16, 4096>;
    using L = BaseCfg<512, 32, 8192>;
    int gs = g_num_sms * 8 * grid_mult, gm = g_num_sms * 4 * grid_mult, gl = g_num_sms * grid_mult;
    unsigned int* cnt = &p.ctrl->n_base[0];
    if (out_f64) {
        k_base<128, 8, 1024, true><<<gs, 128, S::smem, st>>>(p.base[0], cnt + 0, src, out, p.ctrl, p.list_cap);
        k_base<256, 16, 4096, true><<<gm, 256, M::smem, st>>>(p.base[1], cnt + 1, src, out, p.ctrl, p.list_cap);
        k_base<512, 32, 8192, true><<<gl, 512, L::smem, st>>>(p.base[2], cnt + 2, src, out, p.ctrl, p.list_cap);
    } else {
        k_base<128, 8, 1024, false><<<gs, 128, S::smem, st>>>(p.base[0], cnt + 0, src, out, p.ctrl, p.list_cap);
        k_base<256, 16, 4096, false><<<gm, 256, M::smem, st>>>(p.base[1], cnt + 1, src, out, p.ctrl, p.list_cap);
        k_base<512, 32, 8192, false><<<gl, 512, L::smem, st>>>(p.base[2], cnt + 2, src, out, p.ctrl, p.list_cap);
    }
}

void launch_fill(const LevelParams& p, void* out, int out_f64, int grid, cudaStream_t st) {
    if (out_f64) k_fill<true><<<grid, 256, 0, st>>>(p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
    else k_fill<false><<<grid, 256, 0, st>>>(p.fill, &p.ctrl->n_fill, out, p.ctrl, p.list_cap);
}

void launch_small_sort(void* keys, uint64_t n, int f64, uint64_t*, Ctrl* ctrl, cudaStream_t st) {
    using L = BaseCfg<512, 32, 8192>;
    if (f64) k_small_sort<true><<<1, 512, L::smem, st>>>(keys, (uint32_t)n, ctrl);
    else k_small_sort<false><<<1, 512, L::smem, st>>>(keys, (uint32_t)n, ctrl);
}

void launch_classify_ids(const uint8_t* model, const void* keys, uint64_t n, int in_f64, uint32_t* ids,
                         unsigned long long* hist, int payload, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)g_num_sms * 8);
    if (grid < 1) grid = 1;
    size_t sm = sizeof(ModelHdr) + (size_t)payload + 16;
    if (in_f64) k_classify_ids<true><<<grid, 256, sm, st>>>(model, keys, n, ids, hist);
    else k_classify_ids<false><<<grid, 256, sm, st>>>(model, keys, n, ids, hist);
}

void launch_tree_build(const uint64_t* sorted, uint64_t s, uint32_t budget, int eq_mode, uint8_t* model,
                       cudaStream_t st) {
    k_tree_build<<<1, kModelNT, sizeof(ModelSmem), st>>>(sorted, (uint32_t)s, budget, eq_mode, model);
}

void launch_block_sort(uint64_t* keys, uint64_t n, cudaStream_t st) {
    k_block_sort<<<1, kModelNT, sizeof(ModelSmem), st>>>(keys, (uint32_t)n);
}

void launch_verify(const void* keys, uint64_t n, int f64, Ctrl* ctrl, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)g_num_sms * 8);
    if (grid < 1) grid = 1;
    if (f64) k_verify<true><<<grid, 256, 0, st>>>(keys, n, ctrl);
    else k_verify<false><<<grid, 256, 0, st>>>(keys, n, ctrl);
}

void launch_decode(uint64_t* keys, uint64_t n, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)g_num_sms * 8);
    if (grid < 1) grid = 1;
    k_decode<<<grid, 256, 0, st>>>(keys, n);
}

void launch_scatter_mapped(const LevelParams& p, int in_f64, int max_payload, const uint32_t* map,
                           uint32_t nmapped, int grid, cudaStream_t st) {
    if (!p.ntiles) return;
    size_t sm = part_smem_scatter(max_payload, (int)nmapped);
    if (in_f64) k_scatter<true, true><<<grid, kPartNT, sm, st>>>(p, (uint32_t)max_payload, nmapped, map, nmapped);
    else k_scatter<false, true><<<grid, kPartNT, sm, st>>>(p, (uint32_t)max_payload, nmapped, map, nmapped);
}

}  // namespace lsort_dev
