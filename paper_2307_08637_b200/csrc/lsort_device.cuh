// lsort_device.cuh -- device-side building blocks of the B200 LearnedSort.
//
// Key codec, counter-based sampling PRNG, partition-model records and their
// exact per-key classifiers, and block-level primitives (reductions, scans,
// the shared-memory MSD block sort used by the base case and the model
// builder). sm_100a only.
//
// Exactness: every double operation of the reference's per-key model math
// (models.hpp:21,34-43,56-65,162-171) is issued as an explicit
// round-to-nearest intrinsic (__dmul_rn/__dadd_rn/__dsub_rn) so ptxas cannot
// contract a multiply-add into an FMA; the reference is built without FMA
// contraction. Conversions use __ull2double_rn (correctly
// rounded like the host's uint64->double) and truncating casts.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace lsort_dev {

constexpr uint64_t kSign = 0x8000000000000000ull;

#define LSORT_MAX_TREE_DEV 1024   // max SplitterTree budget
#define LSORT_MAX_RMI_DEV 2048    // max RMI submodels / output buckets (shared-memory resident)
constexpr uint32_t kMaxNB = 2048; // max output buckets of any partition model

// keys.hpp:24-27
__device__ __forceinline__ uint64_t encode(double x) {
    // branch-free: negative -> ~b, else b ^ sign  (mask = all ones iff negative)
    const long long b = __double_as_longlong(x);
    return (uint64_t)(b ^ ((b >> 63) | (long long)kSign));
}
// keys.hpp:29-32
__device__ __forceinline__ double decode(uint64_t k) {
    // branch-free inverse: sign bit set -> k ^ sign, else ~k
    const long long b = (long long)k;
    return __longlong_as_double(b ^ ((~b >> 63) | (long long)kSign));
}
// rng.hpp:13-18
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
// Rng(seed).next_below(n) at stream position `draw` (rng.hpp:24,35-37)
__host__ __device__ __forceinline__ uint64_t sample_index(uint64_t seed, uint64_t draw, uint64_t n) {
    return n == 0 ? 0 : splitmix64(seed + draw) % n;
}
// The same index without a 64-bit division (emulated on the GPU, ~100
// instructions): x % n from the high product with minv = floor((2^64-1)/n),
// which underestimates x / n by at most 2 -- exact after two corrections.
__device__ __forceinline__ uint64_t mod_by_inv(uint64_t x, uint64_t n, uint64_t minv) {
    uint64_t r = x - __umul64hi(x, minv) * n;
    r = r >= n ? r - n : r;
    return r >= n ? r - n : r;
}
__device__ __forceinline__ uint64_t sample_index_inv(uint64_t seed, uint64_t draw, uint64_t n, uint64_t minv) {
    return n == 0 ? 0 : mod_by_inv(splitmix64(seed + draw), n, minv);
}

enum ModelKind : uint32_t { kLearned = 0, kTree = 1, kRadix = 2, kFill = 3 };

struct RmiEntry {
    double slope, intercept, lo, hi;
};

// Compiled learned table used by the partition kernels (follows RmiEntry[B]
// in the model record): the submodel line plus the BUCKET ids of its clamp
// bounds. The reference bucket is g(min(max(v, lo), hi)) with
// g = bucket_of o clamp01 monotone nondecreasing (models.hpp:38-41,166-170),
// which equals min(max(h(v), g(lo)), g(hi)) for the unclamped bucket h(v) --
// two integer min/max instead of six double clamps, bit-identical ids.
struct RmiBucketEntry {
    double slope, intercept;
    uint32_t glo, ghi;
    uint64_t pad;
};
constexpr uint32_t kLearnedEntryBytes = sizeof(RmiEntry) + sizeof(RmiBucketEntry);  // 64
constexpr uint32_t kModelIdentityCdf = 1u;  // ModelHdr.flags: cdf_lo == 0 and inv_span == 1
// Cell-table partition model (GPU policy for learned-eligible segments below the
// root, see models.cu build_lut_block): kind kRadix with flags & kModelLut,
// radix_min = origin of the cells, shift = log2 cell width, B = cells; payload
// uint16 lut[B], the bucket of every key of cell c. Monotone: buckets are unions
// of consecutive cells. Classifies with one table read instead of an RMI.
constexpr uint32_t kModelLut = 2u;
constexpr uint32_t kLutModelMaxCells = 8192;
constexpr uint32_t kLutModelCellsPerBucket = 32;
constexpr uint32_t kRootLutCells = 8192;  // a root's table (payload >= 64 B x submodels >= 2 x cells)
// Binade-indexed ("log") cell table for roots whose keys span many binades
// (encoded floats are log-scaled: a linear table over Normal's or a mixture's
// range puts all keys into a few cells). flags kModelLut | kModelLog; radix_min
// = first binade (top 12 key bits) of the table, levels = binades, B = cells;
// payload u16 tab[levels] then u16 lut[B]. tab entry = first cell | log2(cells
// of the binade) << 12 (empty binades: the next binade's first cell, 0 bits).
constexpr uint32_t kModelLog = 4u;
constexpr uint32_t kBinadeCells = 4096, kLogTabMax = 4096;
__device__ __forceinline__ uint32_t binade_cell(uint64_t x, const uint16_t* tab, uint32_t bmin, uint32_t ntab,
                                             uint32_t ncell) {
    const uint32_t hi = (uint32_t)(x >> 32);
    const int bi = (int)(hi >> 20) - (int)bmin;
    const uint32_t e = tab[min(max(bi, 0), (int)ntab - 1)], k = e >> 12;
    const uint32_t c = (e & 0xfffu) + ((hi >> (20 - k)) & ((1u << k) - 1u));
    return bi < 0 ? 0u : (bi >= (int)ntab ? ncell - 1 : c);
}
__host__ __device__ __forceinline__ uint32_t lut_model_cells(uint32_t nb) {
    const uint32_t c = nb * kLutModelCellsPerBucket;
    return c < kLutModelMaxCells ? c : kLutModelMaxCells;
}
// Cell of key x. Narrow tables (shift < 32): cells of 2^shift keys from the
// origin. Wide tables (shift >= 32): cells aligned to multiples of 2^shift, so
// the cell index is a 32-bit function of the key's high word (half the
// instructions of the 64-bit offset); lut_pick_shift makes both fit ncell cells.
__device__ __forceinline__ uint32_t lut_cell(uint64_t x, uint64_t origin, uint32_t shift, uint32_t ncell) {
    if (shift >= 32) {
        const uint32_t h = (uint32_t)(x >> 32) >> (shift - 32), o = (uint32_t)(origin >> shift);
        return h > o ? min(h - o, ncell - 1) : 0u;
    }
    const uint64_t c = (x > origin ? x - origin : 0ull) >> shift;
    return c < ncell ? (uint32_t)c : ncell - 1;
}
// first key of cell c >= 1 (saturating)
__device__ __forceinline__ uint64_t lut_cell_start(uint32_t c, uint64_t origin, uint32_t shift) {
    if (shift >= 32) {
        const uint64_t q = (origin >> shift) + c;
        return q >= (1ull << (64 - shift)) ? ~0ull : q << shift;
    }
    const uint64_t off = (uint64_t)c << shift;
    return off > ~0ull - origin ? ~0ull : origin + off;
}
// smallest shift whose cells over [lo, hi] fit ncell (a power of two)
__device__ __forceinline__ uint32_t lut_pick_shift(uint64_t lo, uint64_t hi, uint32_t ncell) {
    const uint32_t lg = 31 - __clz(ncell);
    const uint32_t bits = hi > lo ? 64u - (uint32_t)__clzll((long long)(hi - lo)) : 0u;
    uint32_t s = bits > lg ? bits - lg : 0u;
    if (s >= 32)
        while (s < 63 && (hi >> s) - (lo >> s) > ncell - 1) ++s;
    return s;
}

// Partition-model record, 128 bytes; payload follows in the model arena:
//   learned: RmiEntry[B]
//   tree:    uint64 tree[leaf_origin], uint64 splitters[nsplit], uint32 eq_offset[nsplit+1]
struct ModelHdr {
    uint32_t kind;       // ModelKind
    uint32_t nbuckets;   // output buckets
    uint32_t B;          // learned: submodels
    uint32_t levels;     // tree
    uint32_t leaf_origin;
    uint32_t nsplit;
    uint32_t shift;      // radix
    uint32_t flags;
    double root_slope, root_icpt, key_base, key_scale;
    double cdf_lo, inv_span;
    uint64_t radix_min;  // radix; fill value for kFill
    double dup;          // duplicate fraction of the first sample
    uint64_t s1, s2;     // sample sizes used
    uint64_t reserved[2];
};
static_assert(sizeof(ModelHdr) == 128, "ModelHdr must stay 128 bytes");

__host__ __device__ __forceinline__ size_t tree_payload_bytes(uint32_t leaf_origin, uint32_t nsplit) {
    return (size_t)leaf_origin * 8 + (size_t)nsplit * 8 + ((size_t)nsplit + 1) * 4;
}

// ---------------------------------------------------------------- classifiers
// Rmi::route (models.hpp:60-65): !(t > 0) -> 0, truncate, clamp to B-1.
// Branch-free: fmax maps t <= 0 and NaN to 0; the saturating truncation and
// min() give B-1 for t >= B -- identical wherever the reference's size_t
// cast is defined (t < 2^64).
// The truncating conversion saturates (negative and NaN -> 0, >= 2^32 -> max),
// which is exactly the reference's !(t > 0) -> 0 plus the clamp.
__device__ __forceinline__ uint32_t rmi_route(double root_slope, double root_icpt, uint32_t B, double xn) {
    double t = __dmul_rn(__dadd_rn(__dmul_rn(root_slope, xn), root_icpt), (double)B);
    return min(__double2uint_rz(t), B - 1);
}

// Clamp of a submodel prediction (models.hpp:38-41): [lo,hi] then [0,1].
// fmax/fmin equal the reference's compare-and-assign for every non-NaN v
// (up to the sign of a zero, which no later step distinguishes: t = v*B is
// only tested with t > 0 and truncated). v is never NaN: xn and the trained
// parameters are finite.
__device__ __forceinline__ double clamp_pred(double v, double lo, double hi) {
    return fmin(fmax(fmin(fmax(v, lo), hi), 0.0), 1.0);
}
// bucket of a CDF value: t = ((f - cdf_lo) * inv_span) * nb, !(t > 0) -> 0,
// truncate, clamp to nb-1 (models.hpp:166-170)
__device__ __forceinline__ uint32_t cdf_bucket(double f, double cdf_lo, double inv_span, uint32_t nb) {
    double t = __dmul_rn(__dmul_rn(__dsub_rn(f, cdf_lo), inv_span), (double)nb);
    return min(__double2uint_rz(t), nb - 1);
}
// g(v) = bucket of clamp01(v) (reference compare-and-assign clamp)
__device__ __forceinline__ uint32_t cdf_bucket_clamped(double v, double cdf_lo, double inv_span, uint32_t nb) {
    if (v < 0.0) v = 0.0;
    if (v > 1.0) v = 1.0;
    return cdf_bucket(v, cdf_lo, inv_span, nb);
}
// Fill the compiled table of a learned model record (header + RmiEntry[B]).
__device__ __forceinline__ void compile_learned(uint8_t* model, uint32_t tid, uint32_t nthreads) {
    ModelHdr* h = (ModelHdr*)model;
    const RmiEntry* E = (const RmiEntry*)(model + sizeof(ModelHdr));
    RmiBucketEntry* C = (RmiBucketEntry*)(model + sizeof(ModelHdr) + sizeof(RmiEntry) * (size_t)h->B);
    for (uint32_t m = tid; m < h->B; m += nthreads) {
        RmiBucketEntry c;
        c.slope = E[m].slope;
        c.intercept = E[m].intercept;
        c.glo = cdf_bucket_clamped(E[m].lo, h->cdf_lo, h->inv_span, h->nbuckets);
        c.ghi = cdf_bucket_clamped(E[m].hi, h->cdf_lo, h->inv_span, h->nbuckets);
        c.pad = 0;
        C[m] = c;
    }
    if (tid == 0) h->flags = (h->cdf_lo == 0.0 && h->inv_span == 1.0) ? kModelIdentityCdf : 0u;
}

// Rmi::normalize (models.hpp:56-58)
__device__ __forceinline__ double rmi_normalize(double key_base, double key_scale, uint64_t x) {
    return __dmul_rn(__dsub_rn(__ull2double_rn(x), key_base), key_scale);
}

// Rmi::predict (models.hpp:34-43)
__device__ __forceinline__ double rmi_predict(const ModelHdr& h, const RmiEntry* e, uint64_t x) {
    double xn = rmi_normalize(h.key_base, h.key_scale, x);
    uint32_t i = rmi_route(h.root_slope, h.root_icpt, h.B, xn);
    RmiEntry s = e[i];
    return clamp_pred(__dadd_rn(__dmul_rn(s.slope, xn), s.intercept), s.lo, s.hi);
}

// PartitionModel::bucket_index, learned branch (models.hpp:162-171)
__device__ __forceinline__ uint32_t learned_bucket(const ModelHdr& h, const RmiEntry* e, uint64_t x) {
    return cdf_bucket(rmi_predict(h, e, x), h.cdf_lo, h.inv_span, h.nbuckets);
}

// SplitterTree::classify (models.hpp:92-101). Returns bucket | (eq << 31).
__device__ __forceinline__ uint32_t tree_bucket(uint32_t levels, uint32_t leaf_origin, uint32_t nsplit,
                                                const uint64_t* tree, const uint64_t* spl,
                                                const uint32_t* eqo, uint64_t x) {
    uint32_t i = 1;
    for (uint32_t l = 0; l < levels; ++l) i = 2 * i + (x > tree[i] ? 1u : 0u);
    uint32_t base = i - leaf_origin;
    uint32_t eq = (base < nsplit) && (eqo[base + 1] - eqo[base] > 1) && (x == spl[base]);
    return (eqo[base] + eq) | (eq << 31);
}

// ------------------------------------------------------------ block helpers
template <int NT>
__device__ __forceinline__ uint64_t block_reduce_min(uint64_t v, uint64_t* red) {
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < NT / 32 ? red[lane] : ~0ull;
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
            v = w < v ? w : v;
        }
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

template <int NT>
__device__ __forceinline__ uint64_t block_reduce_max(uint64_t v, uint64_t* red) {
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < NT / 32 ? red[lane] : 0ull;
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
            v = w > v ? w : v;
        }
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

template <int NT>
__device__ __forceinline__ uint64_t block_reduce_sum_u64(uint64_t v, uint64_t* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < NT / 32 ? red[lane] : 0ull;
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

// Deterministic fixed-order block sum of doubles (tree over lanes, then warps).
template <int NT>
__device__ __forceinline__ double block_sum_f64(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) {
        v = lane < NT / 32 ? red[lane] : 0.0;
        for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

// In-place exclusive scan of a[0,n) (u32) by the whole block; returns total.
// `wsum` needs NT/32 + 1 words.
template <int NT>
__device__ uint32_t block_exclusive_scan_u32(uint32_t* a, uint32_t n, uint32_t* wsum) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t per = (n + NT - 1) / NT;  // contiguous chunk per thread
    const uint32_t lo = threadIdx.x * per;
    const uint32_t hi = min(lo + per, n);
    uint32_t s = 0;
    for (uint32_t i = lo; i < hi; ++i) s += a[i];
    uint32_t incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t w = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += w;
    }
    __syncthreads();
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = lane < NT / 32 ? wsum[lane] : 0;
        uint32_t inc2 = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t w = __shfl_up_sync(0xffffffffu, inc2, o);
            if (lane >= o) inc2 += w;
        }
        if (lane < NT / 32) wsum[lane] = inc2 - v;
        if (lane == NT / 32 - 1) wsum[NT / 32] = inc2;
    }
    __syncthreads();
    uint32_t run = wsum[warp] + incl - s;
    for (uint32_t i = lo; i < hi; ++i) {
        uint32_t t = a[i];
        a[i] = run;
        run += t;
    }
    uint32_t total = wsum[NT / 32];
    __syncthreads();
    return total;
}

// In-place exclusive scan, u64 values.
template <int NT>
__device__ uint64_t block_exclusive_scan_u64(uint64_t* a, uint32_t n, uint64_t* wsum) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t per = (n + NT - 1) / NT;
    const uint32_t lo = threadIdx.x * per;
    const uint32_t hi = min(lo + per, n);
    uint64_t s = 0;
    for (uint32_t i = lo; i < hi; ++i) s += a[i];
    uint64_t incl = s;
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t w = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += w;
    }
    __syncthreads();
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint64_t v = lane < NT / 32 ? wsum[lane] : 0;
        uint64_t inc2 = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t w = __shfl_up_sync(0xffffffffu, inc2, o);
            if (lane >= o) inc2 += w;
        }
        if (lane < NT / 32) wsum[lane] = inc2 - v;
        if (lane == NT / 32 - 1) wsum[NT / 32] = inc2;
    }
    __syncthreads();
    uint64_t run = wsum[warp] + incl - s;
    for (uint32_t i = lo; i < hi; ++i) {
        uint64_t t = a[i];
        a[i] = run;
        run += t;
    }
    uint64_t total = wsum[NT / 32];
    __syncthreads();
    return total;
}

__device__ __forceinline__ uint32_t bitlen64(uint64_t v) { return v ? 64u - (uint32_t)__clzll((long long)v) : 0u; }

// ----------------------------------------------------------- block sort
// Shared-memory sort of up to NT*ITEMS keys (the GPU base case; also sorts
// samples for the model builder). One range-adaptive counting pass buckets
// keys by (k - min) >> shift into ~one key per digit; then every key of a
// digit with <= 16 keys computes its final slot directly (digit start + number
// of smaller keys in its digit, ties by staging index) -- no per-digit
// insertion sort, no divergence. Digits of 17..256 keys are rank-sorted by one
// warp, larger ones get another counting pass (keys re-staged through
// registers; the digit span shrinks by NBMAX each pass, so this terminates
// for any input). Equal-key ranges end at once (min == max).
template <int NT, int ITEMS, int NBMAX>
struct BlockSort {
    static constexpr int CAP = NT * ITEMS;
    static constexpr int kSmall = 16;
    static constexpr int kMedium = 256;
    static constexpr int kListCap = CAP / (kSmall + 1) + 2;
    static_assert(CAP <= 65536, "ranks are packed in 16 bits");
    static constexpr int kRk = (ITEMS + 1) / 2;  // two 16-bit ranks per register
    __device__ static __forceinline__ uint32_t rk_get(const uint32_t (&r)[kRk], int i) {
        return (i & 1) ? (r[i >> 1] >> 16) : (r[i >> 1] & 0xffffu);
    }
    __device__ static __forceinline__ void rk_set(uint32_t (&r)[kRk], int i, uint32_t v) {
        r[i >> 1] = (i & 1) ? ((r[i >> 1] & 0xffffu) | (v << 16)) : ((r[i >> 1] & 0xffff0000u) | v);
    }
    struct Smem {
        uint32_t hist[NBMAX + 1];
        uint32_t wsum[NT / 32 + 1];
        uint64_t red[2 * (NT / 32)];
        uint32_t n_med, n_large;
        uint32_t med[kListCap];
        uint32_t med_len[kListCap];
        uint32_t large[kListCap];
        uint32_t large_len[kListCap];
    };

    // warp rank sort of a[0,len), len <= 256
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
            for (int q = 0; q < 8; ++q) {
                uint32_t idx = lane + 32 * q;
                r[q] += (w < v[q]) || (w == v[q] && j < idx);
            }
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint32_t idx = lane + 32 * q;
            if (idx < len) a[r[q]] = v[q];
        }
        __syncwarp();
    }

    __device__ static __forceinline__ void push_big(Smem& S, uint32_t at, uint32_t l) {
        if (l <= (uint32_t)kMedium) {
            uint32_t q = atomicAdd(&S.n_med, 1u);
            S.med[q] = at;
            S.med_len[q] = l;
        } else {
            uint32_t q = atomicAdd(&S.n_large, 1u);
            S.large[q] = at;
            S.large_len[q] = l;
        }
    }

    // One distribution pass over keys held in registers k[] (valid where
    // idx < len, idx = tid + i*NT), writing the result into a[off, off+len).
    __device__ static __forceinline__ void pass(uint64_t (&k)[ITEMS], uint64_t* a, uint32_t off, uint32_t len,
                                                Smem& S) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        // ---- min and max in one reduction (one barrier)
        uint64_t mn = ~0ull, mx = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = tid + i * NT;
            if (idx < len) {
                mn = k[i] < mn ? k[i] : mn;
                mx = k[i] > mx ? k[i] : mx;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t a1 = __shfl_xor_sync(0xffffffffu, mn, o), b1 = __shfl_xor_sync(0xffffffffu, mx, o);
            mn = a1 < mn ? a1 : mn;
            mx = b1 > mx ? b1 : mx;
        }
        if (lane == 0) { S.red[2 * warp] = mn; S.red[2 * warp + 1] = mx; }
        __syncthreads();
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) {
            uint64_t a1 = S.red[2 * w], b1 = S.red[2 * w + 1];
            mn = a1 < mn ? a1 : mn;
            mx = b1 > mx ? b1 : mx;
        }
        if (mn == mx) {  // homogeneous: write back unchanged
#pragma unroll
            for (int i = 0; i < ITEMS; ++i) {
                uint32_t idx = tid + i * NT;
                if (idx < len) a[off + idx] = k[i];
            }
            __syncthreads();
            return;
        }
        uint32_t nb = 1;  // ~two keys per digit
        while (2 * nb < len && nb < (uint32_t)NBMAX) nb <<= 1;
        const uint32_t lgnb = __ffs(nb) - 1;
        const uint32_t bits = bitlen64(mx - mn);
        const uint32_t shift = bits > lgnb ? bits - lgnb : 0;
        for (uint32_t d = tid; d < nb; d += NT) S.hist[d] = 0;
        __syncthreads();
        uint32_t rank[kRk];
#pragma unroll
        for (int i = 0; i < kRk; ++i) rank[i] = 0;
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = tid + i * NT;
            if (idx < len) rk_set(rank, i, atomicAdd(&S.hist[(uint32_t)((k[i] - mn) >> shift)], 1u));
        }
        __syncthreads();
        // ---- exclusive scan of hist[0,nb) with big-digit detection
        {
            const uint32_t per = (nb + NT - 1) / NT;
            const uint32_t lo = min(nb, tid * per), hi = min(nb, lo + per);
            uint32_t sum = 0;
            for (uint32_t d = lo; d < hi; ++d) sum += S.hist[d];
            uint32_t incl = sum;
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t w = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += w;
            }
            if (lane == 31) S.wsum[warp] = incl;
            __syncthreads();
            uint32_t run = incl - sum;
            for (int w = 0; w < warp; ++w) run += S.wsum[w];
            for (uint32_t d = lo; d < hi; ++d) {
                uint32_t t = S.hist[d];
                S.hist[d] = run;
                if (t > (uint32_t)kSmall) push_big(S, off + run, t);
                run += t;
            }
            if (tid == 0) S.hist[nb] = len;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = tid + i * NT;
            if (idx < len) a[off + S.hist[(uint32_t)((k[i] - mn) >> shift)] + rk_get(rank, i)] = k[i];
        }
        __syncthreads();
        // final slots for keys of small digits (rank within digit)
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = tid + i * NT;
            if (idx < len) {
                const uint32_t d = (uint32_t)((k[i] - mn) >> shift);
                const uint32_t s0 = S.hist[d], c = S.hist[d + 1] - s0, me = s0 + rk_get(rank, i);
                uint32_t p = me;
                if (c <= (uint32_t)kSmall) {
                    p = s0;
                    for (uint32_t j = s0; j < s0 + c; ++j) {
                        const uint64_t w = a[off + j];
                        p += (w < k[i]) || (w == k[i] && j < me);
                    }
                }
                rk_set(rank, i, p);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = tid + i * NT;
            if (idx < len) a[off + rk_get(rank, i)] = k[i];
        }
        __syncthreads();
    }

    // fallback pass over a range already in shared memory (kept out of line)
    __device__ static __noinline__ void pass_smem(uint64_t* a, uint32_t off, uint32_t len, Smem& S) {
        uint64_t k[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            uint32_t idx = threadIdx.x + i * NT;
            if (idx < len) k[i] = a[off + idx];
        }
        __syncthreads();
        pass(k, a, off, len, S);
    }

    // Sort a[0,n) in shared memory; keys arrive in registers k[] (idx = tid + i*NT).
    __device__ static void sort_regs(uint64_t (&k)[ITEMS], uint64_t* a, uint32_t n, Smem& S) {
        if (threadIdx.x == 0) {
            S.n_med = 0;
            S.n_large = 0;
        }
        __syncthreads();
        pass(k, a, 0, n, S);
        if (S.n_med | S.n_large) finish(a, S);
    }

    __device__ static __noinline__ void finish(uint64_t* a, Smem& S) {
        const int warp = threadIdx.x >> 5;
        for (;;) {
            uint32_t nm = S.n_med;
            uint32_t nl = S.n_large;
            if (nm == 0 && nl == 0) break;
            for (uint32_t e = warp; e < nm; e += NT / 32) warp_rank_sort(a + S.med[e], S.med_len[e]);
            __syncthreads();
            if (threadIdx.x == 0) S.n_med = 0;
            if (nl == 0) {
                __syncthreads();
                break;
            }
            uint32_t off = S.large[nl - 1], len = S.large_len[nl - 1];
            __syncthreads();
            if (threadIdx.x == 0) S.n_large = nl - 1;
            pass_smem(a, off, len, S);
        }
    }
};

}  // namespace lsort_dev
