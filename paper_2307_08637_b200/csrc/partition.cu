// partition.cu -- one distribution level: classify + histogram, per-segment
// scan, and the shared-memory staged scatter.
//
//   k_kind_plan      compacts the level's segments by partition-model kind
//                    (learned / tree / radix) and builds per-kind tile prefixes,
//                    so each kind runs a specialised kernel over a balanced
//                    tile range (no per-key kind dispatch, no register spill).
//   k_hist<K>        fused decode/encode + model inference + shared-memory
//                    histogram (hardware-aggregated atomics, see hist_add);
//                    8 keys per thread read from TMA tiles, persistent; the
//                    bucket id of every key is stored (u16, 2 B/key) so the
//                    scatter does not classify again.
//   k_scan_children  per-segment exclusive scan -> write cursors; emits base
//                    case / equality fill / recursion work lists.
//   k_scatter        one kernel for all model kinds: read keys + ids, rank
//                    within the tile, claim one range per bucket per tile
//                    (global atomic), stage the tile grouped by bucket in
//                    shared memory, write each bucket run coalesced.
//
// Model tables (learned: 20 B per submodel; tree payload) are copied to
// shared memory by k_hist.
#include <algorithm>
#include <climits>

#include "kernels_common.cuh"
#include "tma.cuh"

namespace lsort_dev {

constexpr int kPNT = kPartNT;             // threads per partition CTA
constexpr int kPItems = 8;                // keys per thread per tile
constexpr int kPPairs = kPItems / 2;      // 128-bit loads per thread per tile
static_assert(kPNT * kPItems == kTileKeys, "tile geometry");

__device__ __forceinline__ uint32_t kind_slot(uint32_t kind) {
    return kind == kLearned ? 0u : (kind == kTree ? 1u : 2u);
}

// one-pass level 1 over part of a level (LevelParams::seg_sel)
__device__ __forceinline__ bool seg_selected(const LevelParams& p, uint32_t i) {
    return p.seg_sel == 0 || (p.seg_direct[i] != 0) == (p.seg_sel == 1);
}

// ------------------------------------------------------------ kind plan
constexpr int kPlanNT = 1024;
__global__ void __launch_bounds__(kPlanNT) k_kind_plan(LevelParams p) {
    griddep_wait();
    if (p.gate && *p.gate == 0) {
        if (threadIdx.x < 3) { p.kplan[threadIdx.x].nsegs = 0; p.kplan[threadIdx.x].ntiles = 0; }
        return;
    }
    __shared__ uint32_t wsum[kPlanNT / 32 + 1];
    __shared__ uint64_t wsum64[kPlanNT / 32 + 1];
    __shared__ uint32_t fl[kPlanNT];
    __shared__ uint64_t tl[kPlanNT];
    __shared__ uint32_t carry_n;
    __shared__ uint64_t carry_t;
    const uint32_t nlists = p.seg_sel == 2 ? 4u : 3u;  // (slot 3: every selected segment, for k_scatter)
    for (uint32_t K = 0; K < nlists; ++K) {
        if (threadIdx.x == 0) { carry_n = 0; carry_t = 0; }
        __syncthreads();
        uint32_t* ks = p.kseg + (size_t)K * p.kstride;
        uint64_t* tp = p.ktp + (size_t)K * (p.kstride + 1);
        for (uint32_t base = 0; base < p.nsegs; base += kPlanNT) {
            uint32_t s = base + threadIdx.x;
            uint32_t f = 0;
            uint64_t t = 0;
            if (s < p.nsegs && seg_selected(p, s)) {
                const SegDesc& sd = p.segs[s];
                uint32_t kind = ((const ModelHdr*)(p.models + sd.model_off))->kind;
                f = K == 3 || kind_slot(kind) == K;
                t = f ? (sd.n + kTileKeys - 1) / kTileKeys : 0;
            }
            fl[threadIdx.x] = f;
            tl[threadIdx.x] = t;
            __syncthreads();
            uint32_t tot = block_exclusive_scan_u32<kPlanNT>(fl, kPlanNT, wsum);
            uint64_t tott = block_exclusive_scan_u64<kPlanNT>(tl, kPlanNT, wsum64);
            if (f) {
                ks[carry_n + fl[threadIdx.x]] = s;
                tp[carry_n + fl[threadIdx.x]] = carry_t + tl[threadIdx.x];
            }
            __syncthreads();
            if (threadIdx.x == 0) { carry_n += tot; carry_t += tott; }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            tp[carry_n] = carry_t;
            p.kplan[K].nsegs = carry_n;
            p.kplan[K].ntiles = carry_t;
        }
        __syncthreads();
    }
}

// ------------------------------------------------------ per-kind models
// Registers-resident model state; tree payload lives in shared memory.
struct KState {
    // learned
    double rs, ri, base, scale, cdf_lo, inv_span;
    const double2* line;      // shared: {slope, intercept} per submodel
    const uint32_t* gbounds;  // shared: g(lo) | g(hi) << 16 per submodel
    uint32_t B, nb, identity;
    // tree (shared memory)
    const uint64_t* tree;
    const uint64_t* spl;
    const uint32_t* eqo;
    uint32_t levels, leaf, nsplit;
    // radix-assisted tree lookup: lut[c] = #splitters below the start of cell c of
    // the splitter range (cells of 2^lshift keys); rank search of <= lutT steps
    const uint16_t* lut;
    uint64_t lbase;
    uint32_t lshift, lutT, llog;
    // radix / fill / cell table (rlut: shared memory, rcells entries; nullptr = plain radix)
    uint64_t rmin;
    uint32_t shift, fill, rcells;
    const uint16_t* rlut;
    uint32_t rorg;  // wide cell tables: (rmin >> shift), the high-word origin (lut_cell)
    const uint16_t* rtab;  // log tables: binade entries (shared), nullptr otherwise
    uint32_t rtabn;
};

// tree payload capacity (tree_payload_bytes(1024, 1023), 16-byte rounded)
constexpr size_t kTreeCapBytes =
    ((size_t)LSORT_MAX_TREE_DEV * 8 + (size_t)(LSORT_MAX_TREE_DEV - 1) * 8 + (size_t)LSORT_MAX_TREE_DEV * 4 + 15) & ~(size_t)15;
constexpr int kLutBits = 12;
constexpr uint32_t kLutCells = 1u << kLutBits;
constexpr uint32_t kLutMaxT = 4;  // longer in-cell searches: descend the tree instead
constexpr size_t kLutBytes = 2 * (kLutCells + 2);
// Log-spaced cells (skewed splitters, e.g. Zipf ranks): offsets r < 64 get a cell
// each, then every octave [2^e, 2^(e+1)) is split into 64 equal cells.
constexpr uint32_t kLogSub = 6;
__device__ __forceinline__ uint32_t log_cell(uint64_t r) {
    if (r < (1ull << kLogSub)) return (uint32_t)r;
    const uint32_t e = 63 - __clzll((long long)r);
    return ((e - kLogSub + 1) << kLogSub) | (uint32_t)((r >> (e - kLogSub)) & ((1u << kLogSub) - 1));
}
__device__ __forceinline__ uint64_t log_cell_start(uint32_t c) {
    if (c < (1u << kLogSub)) return c;
    const uint32_t k = c >> kLogSub, low = c & ((1u << kLogSub) - 1);
    return ((1ull << kLogSub) + low) << (k - 1);
}
constexpr uint32_t kLogCells = (64 - kLogSub + 1) << kLogSub;  // 3776 <= kLutCells
static_assert(kLogCells <= kLutCells, "log cells fit the table");

// #{i < n : a[i] < x} over a strictly increasing array
__device__ __forceinline__ uint32_t lower_rank(const uint64_t* a, uint32_t n, uint64_t x) {
    uint32_t b = 0;
    while (n > 0) {
        const uint32_t h = n >> 1;
        if (a[b + h] < x) { b += h + 1; n -= h + 1; }
        else n = h;
    }
    return b;
}

template <uint32_t KIND>
__device__ __forceinline__ void kstate_load(KState& S, const uint8_t* g, uint8_t* tree_smem,
                                            uint16_t* lut_smem = nullptr, uint32_t* red = nullptr) {
    const ModelHdr* h = (const ModelHdr*)g;
    S.nb = h->nbuckets;
    if constexpr (KIND == kLearned) {
        // compiled table -> shared memory (20 B per submodel): the L1 cannot be
        // relied on once the TMA tile buffers take most of the SM's shared memory
        S.rs = h->root_slope; S.ri = h->root_icpt; S.base = h->key_base; S.scale = h->key_scale;
        S.cdf_lo = h->cdf_lo; S.inv_span = h->inv_span; S.B = h->B;
        S.identity = h->flags & kModelIdentityCdf;
        const RmiBucketEntry* E = (const RmiBucketEntry*)(g + sizeof(ModelHdr) + sizeof(RmiEntry) * (size_t)S.B);
        double2* line = (double2*)tree_smem;
        uint32_t* gbounds = (uint32_t*)(line + S.B);
        __syncthreads();  // previous users of the table are done
        for (uint32_t m = threadIdx.x; m < S.B; m += blockDim.x) {
            const RmiBucketEntry e = E[m];
            line[m] = make_double2(e.slope, e.intercept);
            gbounds[m] = e.glo | (e.ghi << 16);
        }
        S.line = line;
        S.gbounds = gbounds;
        __syncthreads();
    } else if constexpr (KIND == kTree) {
        S.levels = h->levels; S.leaf = h->leaf_origin; S.nsplit = h->nsplit;
        uint32_t words = (uint32_t)((tree_payload_bytes(S.leaf, S.nsplit) + 15) / 16);
        const uint4* src = (const uint4*)(g + sizeof(ModelHdr));
        __syncthreads();  // previous users of tree_smem are done
        for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) ((uint4*)tree_smem)[i] = src[i];
        S.tree = (const uint64_t*)tree_smem;
        S.spl = S.tree + S.leaf;
        S.eqo = (const uint32_t*)(S.spl + S.nsplit);
        S.lutT = ~0u;
        __syncthreads();
        if (lut_smem && S.nsplit >= 8) {
            // the tree's leaf is the splitters' lower rank (padding is UINT64_MAX,
            // models.cpp:133-185): index a cell of the splitter range, then search
            // the few splitters inside it
            const uint64_t s0 = S.spl[0], range = S.spl[S.nsplit - 1] - s0;
            const int bl = 64 - __clzll((long long)range);
            S.lbase = s0;
            S.lshift = bl > kLutBits ? (uint32_t)(bl - kLutBits) : 0u;
            for (uint32_t mode = 0; mode < 2 && S.lutT == ~0u; ++mode) {  // linear cells, then log cells
                const uint32_t ncell = mode ? kLogCells : kLutCells;
                if (threadIdx.x == 0) *red = 0;
                for (uint32_t c = threadIdx.x; c <= ncell; c += blockDim.x) {
                    uint32_t r = S.nsplit;
                    if (c < ncell) {
                        const uint64_t off = mode ? log_cell_start(c) : (uint64_t)c << S.lshift;
                        const uint64_t start = off > ~0ull - s0 ? ~0ull : s0 + off;
                        r = lower_rank(S.spl, S.nsplit, start);
                    }
                    lut_smem[c] = (uint16_t)r;
                }
                __syncthreads();
                uint32_t mx = 0;
                for (uint32_t c = threadIdx.x; c < ncell; c += blockDim.x)
                    mx = max(mx, (uint32_t)lut_smem[c + 1] - lut_smem[c]);
                for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
                if ((threadIdx.x & 31) == 0 && mx) atomicMax(red, mx);
                __syncthreads();
                const uint32_t T = 32 - __clz(*red);  // steps of a lower-bound search over <= max keys
                S.lutT = T <= kLutMaxT ? T : ~0u;
                S.llog = mode;
                __syncthreads();  // *red and the table are reused by the next mode
            }
            S.lut = lut_smem;
        }
    } else {
        S.rmin = h->radix_min; S.shift = h->shift; S.fill = h->kind == kFill;
        S.rlut = nullptr;
        S.rcells = h->B;
        S.rorg = S.shift >= 32 ? (uint32_t)(S.rmin >> S.shift) : 0u;
        S.rtab = nullptr;
        S.rtabn = h->levels;
        if (h->kind == kRadix && (h->flags & kModelLut)) {  // the cell table (log: binade entries first) -> shared memory
            const uint4* src = (const uint4*)(g + sizeof(ModelHdr));
            const bool lg = h->flags & kModelLog;
            const uint32_t tabw = lg ? (2 * S.rtabn + 15) / 16 : 0u;
            const uint32_t words = tabw + (2 * S.rcells + 15) / 16;
            __syncthreads();  // previous users of tree_smem are done
            for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) ((uint4*)tree_smem)[i] = src[i];
            if (lg) S.rtab = (const uint16_t*)tree_smem;
            S.rlut = (const uint16_t*)tree_smem + 8 * tabw;
            __syncthreads();
        }
    }
}

// bucket id | (eq << 31): bit-exact learned math of models.hpp:34-43,162-171
template <uint32_t KIND>
__device__ __forceinline__ uint32_t kclassify(const KState& S, uint64_t x) {
    if constexpr (KIND == kLearned) {
        // models.hpp:34-43,56-65,162-171 via the compiled table (RmiBucketEntry)
        const double xn = rmi_normalize(S.base, S.scale, x);
        const uint32_t m = rmi_route(S.rs, S.ri, S.B, xn);
        const double2 li = S.line[m];
        const uint32_t gb = S.gbounds[m];
        const double v = __dadd_rn(__dmul_rn(li.x, xn), li.y);
        // one formula for every model: with the identity range (cdf_lo 0, inv_span 1)
        // the subtraction and the first product are exact, so t == v * nb bit for bit
        // (no per-key select between two paths)
        const double t = __dmul_rn(__dmul_rn(__dsub_rn(v, S.cdf_lo), S.inv_span), (double)S.nb);
        // g(hi) <= nb - 1, so the clamp to nb - 1 is implied by the last min
        return min(max(__double2uint_rz(t), gb & 0xffffu), gb >> 16);
    } else if constexpr (KIND == kTree) {
        return tree_bucket(S.levels, S.leaf, S.nsplit, S.tree, S.spl, S.eqo, x);
    } else {
        if (S.fill) return 1u << 31;
        if (S.rlut) {  // lut_cell with the origin's high word precomputed
            if (S.rtab) return S.rlut[binade_cell(x, S.rtab, (uint32_t)S.rmin, S.rtabn, S.rcells)];
            if (S.shift >= 32) {
                const uint32_t h = (uint32_t)(x >> 32) >> (S.shift - 32);
                return S.rlut[h > S.rorg ? min(h - S.rorg, S.rcells - 1) : 0u];
            }
            return S.rlut[lut_cell(x, S.rmin, S.shift, S.rcells)];
        }
        uint64_t d = (x - S.rmin) >> S.shift;
        return d >= S.nb ? S.nb - 1 : (uint32_t)d;
    }
}

template <uint32_t KIND>
struct KindTiles {
    uint32_t K, nks;
    uint64_t ntiles;
    const uint32_t* ks;
    const uint64_t* tp;
    __device__ __forceinline__ void init(const LevelParams& p) {
        K = kind_slot(KIND);
        nks = p.kplan[K].nsegs;
        ntiles = p.kplan[K].ntiles;
        ks = p.kseg + (size_t)K * p.kstride;
        tp = p.ktp + (size_t)K * (p.kstride + 1);
    }
};

// Classify the 16 keys a thread holds (8 pairs). Trees descend in lockstep
// (16 independent shared-memory loads in flight per level instead of one
// dependent chain per key); learned/radix keys are straight-line code.
template <uint32_t KIND>
__device__ __forceinline__ void classify16(const KState& S, const ulonglong2 (&v)[kPPairs], uint32_t (&c)[kPItems]) {
    if constexpr (KIND == kTree) {
        uint32_t idx[kPItems];
        if (S.lutT != ~0u) {  // radix-assisted: cell lookup + a short lockstep search
            uint32_t n[kPItems];
#pragma unroll
            for (int q = 0; q < kPItems; ++q) {
                const uint64_t x = (q & 1) ? v[q >> 1].y : v[q >> 1].x;
                const uint64_t rel = x < S.lbase ? 0ull : x - S.lbase;
                const uint32_t d = S.llog ? log_cell(rel) : (uint32_t)min(rel >> S.lshift, (uint64_t)(kLutCells - 1));
                const uint32_t b = S.lut[d];
                idx[q] = b;
                n[q] = S.lut[d + 1] - b;
            }
            for (uint32_t it = 0; it < S.lutT; ++it) {
#pragma unroll
                for (int q = 0; q < kPItems; ++q) {
                    const uint64_t x = (q & 1) ? v[q >> 1].y : v[q >> 1].x;
                    const uint32_t h = n[q] >> 1;
                    const bool lt = n[q] > 0 && S.spl[min(idx[q] + h, S.nsplit - 1)] < x;
                    idx[q] = lt ? idx[q] + h + 1 : idx[q];
                    n[q] = lt ? n[q] - h - 1 : h;
                }
            }
#pragma unroll
            for (int q = 0; q < kPItems; ++q) idx[q] += S.leaf;
        } else {
#pragma unroll
            for (int q = 0; q < kPItems; ++q) idx[q] = 1;
            for (uint32_t l = 0; l < S.levels; ++l) {
#pragma unroll
                for (int q = 0; q < kPItems; ++q) {
                    const uint64_t x = (q & 1) ? v[q >> 1].y : v[q >> 1].x;
                    idx[q] = 2 * idx[q] + (x > S.tree[idx[q]] ? 1u : 0u);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < kPItems; ++q) {
            const uint64_t x = (q & 1) ? v[q >> 1].y : v[q >> 1].x;
            const uint32_t base = idx[q] - S.leaf;
            const uint32_t e0 = S.eqo[base];
            const uint32_t eq = (base < S.nsplit) && (S.eqo[base + 1] - e0 > 1) && (x == S.spl[base]);
            c[q] = (e0 + eq) | (eq << 31);
        }
    } else if (KIND == kRadix && S.rlut && !S.rtab && S.shift >= 32) {  // wide cell table: 32-bit cells (lut_cell)
        const uint32_t sh = S.shift - 32, last = S.rcells - 1;
#pragma unroll
        for (int q = 0; q < kPItems; ++q) {
            const uint32_t h = (uint32_t)(((q & 1) ? v[q >> 1].y : v[q >> 1].x) >> 32) >> sh;
            c[q] = S.rlut[h > S.rorg ? min(h - S.rorg, last) : 0u];
        }
    } else {
#pragma unroll
        for (int q = 0; q < kPItems; ++q) c[q] = kclassify<KIND>(S, (q & 1) ? v[q >> 1].y : v[q >> 1].x);
    }
}

// Tile t of a kind list: its segment (index into the kind list) and geometry.
template <uint32_t KIND>
// i: the segment of the previous tile of this CTA (tiles ascend), or ~0 for
// a binary search -- a CTA walks its contiguous tile range, so the segment
// index only ever advances (no dependent search chain per tile).
__device__ __forceinline__ TileGeom tile_geom(const LevelParams& p, const KindTiles<KIND>& KT, uint64_t t,
                                              uint32_t& i) {
    if (i == ~0u) i = find_seg(KT.tp, KT.nks, t);
    else
        while (i + 1 < KT.nks && KT.tp[i + 1] <= t) ++i;
    const SegDesc& sd = p.segs[KT.ks[i]];
    const uint64_t lo = sd.in_begin + (t - KT.tp[i]) * (uint64_t)kTileKeys;
    TileGeom g;
    g.init(p.src, lo, min(lo + kTileKeys, sd.in_begin + sd.n));
    return g;
}

// Double-buffered TMA tile stream: the 16-byte aligned interior of tile t is
// bulk-copied (cp.async.bulk + mbarrier) into shared buffer (t - t0) & 1
// while the previous tile is processed; head/tail singles are read directly.
struct TileStream {
    uint8_t* base;      // two buffers of kTileKeys keys
    uint64_t* bar;      // 2 mbarriers
    uint32_t phase;     // bit b: parity of buffer b's next completion (flips only when a copy was issued)
    __device__ __forceinline__ void init(uint8_t* b, uint64_t* bars) {
        base = b;
        bar = bars;
        phase = 0;
        if (threadIdx.x == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
        }
        __syncthreads();
    }
    // (arithmetic addressing: a runtime-indexed member array would live in local memory)
    __device__ __forceinline__ ulonglong2* buf(int b) const {
        return (ulonglong2*)(base + (size_t)b * (8 * (size_t)kTileKeys));
    }
    __device__ __forceinline__ void issue(const void* src, const TileGeom& g, int b) {
        if (threadIdx.x == 0 && g.npairs) {
            mbar_expect_tx(bar + b, g.npairs * 16);
            tma_load_1d(buf(b), (const uint64_t*)src + g.a0, g.npairs * 16, bar + b);
        }
    }
    // g.npairs is uniform across the CTA, so every thread flips the same bits
    __device__ __forceinline__ void wait(const TileGeom& g, int b) {
        if (g.npairs) {
            mbar_wait(bar + b, (phase >> b) & 1u);
            phase ^= 1u << b;
        }
    }
};
constexpr size_t kTileBytes = 8 * (size_t)kTileKeys;

// ------------------------------------------------------- classify + hist
template <bool IN_F64, uint32_t KIND>
__global__ void __launch_bounds__(kPNT, kPartPerSM) k_hist(LevelParams p) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    uint8_t* sm = (uint8_t*)smem_u4;
    uint64_t* bars = (uint64_t*)sm;                          // 2 mbarriers (16 B)
    uint32_t* hist = (uint32_t*)(sm + 16);                   // kMaxNB
    uint8_t* tiles = sm + 16 + 4 * kMaxNB;                   // 2 x kTileBytes
    uint8_t* tree_smem = tiles + 2 * kTileBytes;             // tree payload (+ lookup table)
    __shared__ uint32_t lut_red;
    if (!IN_F64 && p.ctrl->nan_index != ~0ull) return;
    KindTiles<KIND> KT;
    KT.init(p);
    if (KT.ntiles == 0) return;
    const uint64_t per = (KT.ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * per;
    const uint64_t t1 = min(t0 + per, KT.ntiles);
    if (t0 >= t1) return;
    for (uint32_t b = threadIdx.x; b < kMaxNB; b += kPNT) hist[b] = 0;
    TileStream TS;
    TS.init(tiles, bars);
    uint32_t inext = ~0u;
    TileGeom gnext = tile_geom<KIND>(p, KT, t0, inext);
    TS.issue(p.src, gnext, 0);
    int64_t cur = -1;
    KState S;
    uint64_t boff = 0;
    for (uint64_t tile = t0; tile < t1; ++tile) {
        const int b = (int)((tile - t0) & 1);
        const uint32_t i = inext;
        const TileGeom g = gnext;
        if (tile + 1 < t1) {  // prefetch the next tile into the other buffer
            gnext = tile_geom<KIND>(p, KT, tile + 1, inext);
            TS.issue(p.src, gnext, b ^ 1);
        }
        if ((int64_t)i != cur) {
            if (cur >= 0) {
                __syncthreads();
                for (uint32_t q = threadIdx.x; q < S.nb; q += kPNT) {
                    uint32_t c = hist[q];
                    if (c) { atomicAdd(&p.buckets[boff + q], (unsigned long long)c); hist[q] = 0; }
                }
            }
            const SegDesc& sd = p.segs[KT.ks[i]];
            boff = sd.bucket_off;
            kstate_load<KIND>(S, p.models + sd.model_off, tree_smem, (uint16_t*)(tree_smem + kTreeCapBytes), &lut_red);
            __syncthreads();
            cur = i;
        }
        TS.wait(g, b);
        const ulonglong2* sp = TS.buf(b);
        ulonglong2 v[kPPairs];
#pragma unroll
        for (int j = 0; j < kPPairs; ++j) {
            uint32_t q = threadIdx.x + j * kPNT;
            v[j] = q < g.npairs ? sp[q] : make_ulonglong2(0, 0);
        }
        if (IN_F64) {
            // NaN (keys.hpp:34-42): one predicate OR per key, the exact index only
            // in the (never taken on clean input) slow path
            bool anynan = false;
#pragma unroll
            for (int j = 0; j < kPPairs; ++j)
                anynan |= isnan(__longlong_as_double((long long)v[j].x)) | isnan(__longlong_as_double((long long)v[j].y));
            if (anynan) {
#pragma unroll
                for (int j = 0; j < kPPairs; ++j) {
                    uint32_t q = threadIdx.x + j * kPNT;
                    if (q < g.npairs) {
                        if (isnan(__longlong_as_double((long long)v[j].x)))
                            atomicMin(&p.ctrl->nan_index, (unsigned long long)(g.a0 + 2 * q));
                        if (isnan(__longlong_as_double((long long)v[j].y)))
                            atomicMin(&p.ctrl->nan_index, (unsigned long long)(g.a0 + 2 * q + 1));
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < kPPairs; ++j) {
                v[j].x = encode(__longlong_as_double((long long)v[j].x));
                v[j].y = encode(__longlong_as_double((long long)v[j].y));
            }
        }
        uint32_t code[kPItems];
        classify16<KIND>(S, v, code);
#pragma unroll
        for (int q = 0; q < kPItems; ++q)
            hist_add(hist, code[q] & 0x7fffffffu, threadIdx.x + (q >> 1) * kPNT < g.npairs);
        {  // bucket ids for the scatter (pairs start at an even index iff src is 16 B aligned)
            const bool al = !(g.a0 & 1);
#pragma unroll
            for (int j = 0; j < kPPairs; ++j) {
                const uint32_t qq = threadIdx.x + j * kPNT;
                if (qq < g.npairs) {
                    const uint32_t i0 = (code[2 * j] >> 31) ? kNoMove : code[2 * j];
                    const uint32_t i1 = (code[2 * j + 1] >> 31) ? kNoMove : code[2 * j + 1];
                    uint16_t* d = p.ids + g.a0 + 2 * qq;
                    if (al) *(uint32_t*)d = i0 | (i1 << 16);
                    else { d[0] = (uint16_t)i0; d[1] = (uint16_t)i1; }
                }
            }
        }
        if (threadIdx.x < g.nsingle) {
            uint64_t ix = g.single(threadIdx.x);
            uint64_t k = ((const uint64_t*)p.src)[ix];
            if (IN_F64) {
                double d = __longlong_as_double((long long)k);
                if (isnan(d)) atomicMin(&p.ctrl->nan_index, (unsigned long long)ix);
                k = encode(d);
            }
            const uint32_t c = kclassify<KIND>(S, k);
            atomicAdd(&hist[c & 0x7fffffffu], 1u);
            p.ids[ix] = (c >> 31) ? kNoMove : (uint16_t)c;
        }
        __syncthreads();  // buffer b is free for the tile after next
    }
    for (uint32_t q = threadIdx.x; q < S.nb; q += kPNT) {
        uint32_t c = hist[q];
        if (c) atomicAdd(&p.buckets[boff + q], (unsigned long long)c);
    }
}

// ---------------------------------------------------------- scan children
// One CTA per segment: exclusive scan of the bucket counts -> write cursors;
// children become fill / base-case / recursion work items. The list appends
// are aggregated per CTA (one global atomic per list per round instead of one
// per child: ~32K children hammered the same counters at level 1).
template <int NT>
__global__ void __launch_bounds__(NT) k_scan_children(LevelParams p) {
    griddep_wait();
    __shared__ uint64_t wsum[NT / 32 + 1];
    __shared__ uint32_t lcount[5];             // fill, base0, base1, base2, rec
    __shared__ unsigned long long lkeys[3];    // keys: fill, base, rec
    __shared__ uint32_t gbase[5];
    extern __shared__ uint64_t dyn[];           // cnt[nb], eqval[nb], iseq[nb] (u8)
    if (p.ctrl->nan_index != ~0ull) return;
    if (p.gate && *p.gate == 0) return;
    if (!seg_selected(p, blockIdx.x)) return;  // (its children come from the one-pass level)
    const SegDesc sd = p.segs[blockIdx.x];
    const uint8_t* mg = p.models + sd.model_off;
    const ModelHdr h = *(const ModelHdr*)mg;
    const uint32_t nb = h.nbuckets;
    uint64_t* cnt = dyn;
    uint64_t* eqval = dyn + sd.nb_max;
    uint8_t* iseq = (uint8_t*)(dyn + 2 * (size_t)sd.nb_max);
    for (uint32_t b = threadIdx.x; b < nb; b += NT) {
        cnt[b] = p.buckets[sd.bucket_off + b];
        iseq[b] = 0;
    }
    __syncthreads();
    if (h.kind == kTree) {
        MView m = model_view(mg);
        for (uint32_t i = threadIdx.x; i < h.nsplit; i += NT) {
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
    block_exclusive_scan_u64<NT>(cnt, nb, wsum);
    for (uint32_t b0 = 0; b0 < nb; b0 += NT) {  // CTA-uniform rounds
        const uint32_t b = b0 + threadIdx.x;
        int cls = -1;  // 0 fill, 1..3 base class, 4 rec
        uint64_t begin = 0, len = 0;
        if (threadIdx.x < 5) lcount[threadIdx.x] = 0;
        if (threadIdx.x < 3) lkeys[threadIdx.x] = 0;
        __syncthreads();
        if (b < nb) {
            const uint64_t start = cnt[b];
            const uint64_t end = (b + 1 < nb) ? cnt[b + 1] : sd.n;
            len = end - start;
            begin = sd.begin + start;
            p.buckets[sd.bucket_off + b] = begin;  // write cursor
            if (len) {
                if (iseq[b]) cls = 0;
                else if (len <= p.base_cap[2]) cls = 1 + (len <= p.base_cap[0] ? 0 : (len <= p.base_cap[1] ? 1 : 2));
                else cls = 4;
            }
        }
        // warp-aggregated: one shared atomic per class and per key counter per warp
        // (a thousand lanes on one shared address serialise)
        uint32_t li = 0;
        const int lane = threadIdx.x & 31;
        const unsigned lt = (1u << lane) - 1u;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            const unsigned m = __ballot_sync(FULL_MASK, cls == c);
            if (m) {
                const int leader = __ffs(m) - 1;
                uint32_t base = 0;
                if (lane == leader) base = atomicAdd(&lcount[c], (uint32_t)__popc(m));
                base = __shfl_sync(FULL_MASK, base, leader);
                if (cls == c) li = base + __popc(m & lt);
            }
        }
#pragma unroll
        for (int gk = 0; gk < 3; ++gk) {
            const int grp = cls < 0 ? -1 : (cls == 0 ? 0 : (cls == 4 ? 2 : 1));
            unsigned long long v = grp == gk ? (unsigned long long)len : 0ull;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
            if (lane == 0 && v) atomicAdd(&lkeys[gk], v);
        }
        __syncthreads();
        if (threadIdx.x < 5) {
            const uint32_t c = lcount[threadIdx.x];
            unsigned int* ctr = threadIdx.x == 0 ? &p.ctrl->n_fill
                                : (threadIdx.x == 4 ? &p.ctrl->n_rec : &p.ctrl->n_base[threadIdx.x - 1]);
            gbase[threadIdx.x] = c ? atomicAdd(ctr, c) : 0u;
        }
        if (threadIdx.x < 3 && lkeys[threadIdx.x]) {
            unsigned long long* kc = threadIdx.x == 0 ? &p.ctrl->keys_fill
                                     : (threadIdx.x == 1 ? &p.ctrl->keys_base : &p.ctrl->keys_rec);
            atomicAdd(kc, lkeys[threadIdx.x]);
        }
        __syncthreads();
        if (cls >= 0) {
            const unsigned e = gbase[cls] + li;
            if (cls == 0) {
                if (e < p.list_cap) p.fill[e] = FillItem{begin, len, eqval[b], 0};
                else atomicOr(&p.ctrl->err, 1u);
            } else if (cls < 4) {
                if (e < p.list_cap) p.base[cls - 1][e] = BaseItem{begin, len, (int64_t)begin};
                else atomicOr(&p.ctrl->err, 2u);
            } else {
                const uint32_t depth = sd.depth + 1;
                const uint32_t flags = (len == sd.n || depth > p.depth_cap) ? kSegForceRadix : 0u;
                uint64_t ps = 0;
                if (p.slices && h.kind != kTree) {  // (a tree root's offsets index its first sample)
                    const uint32_t o = p.slices[b], l = p.slices[b + 1] - o;
                    if (l >= kMinSlice) ps = (uint64_t)o << 24 | min(l, 0xffffffu);
                }
                // (read position relative to the next level's source: rec_delta when this
                // level's one-pass part made that source the padded buffer)
                if (e < p.list_cap) p.rec[e] = SegOut{begin, len, depth, flags, ps, (uint64_t)((int64_t)begin + p.rec_delta)};
                else atomicOr(&p.ctrl->err, 4u);
            }
        }
    }
}

// ---------------------------------------------------------------- scatter
// Shared-memory layout at compile-time offsets (NBC = bucket capacity per
// segment): no runtime pointer arithmetic to keep live or rematerialise.
template <uint32_t NBC>
struct ScatterSmem {
    uint64_t bars[2];
    ulonglong2 tiles[2][kTileKeys / 2];  // TMA tile buffers; the consumed one stages the tile
    long long delta[NBC];                // per bucket: claimed global position - tile-local start
    alignas(16) uint32_t cnt[2][NBC + 4];  // per tile parity: counts -> tile-local starts
    uint16_t sbid[kTileKeys];
    uint32_t wsum[kPNT / 32 + 1];
    alignas(16) uint16_t sids[2][kTileKeys + 16];  // the tile's bucket ids, bulk-copied with its keys
};

// ids of a tile's 16-byte interior: the covering 16-byte aligned range of the
// u16 id array (ids [a0 & ~7, roundup8(a0 + 2 npairs)))
__device__ __forceinline__ void ids_range(const TileGeom& g, uint64_t& start, uint32_t& bytes) {
    start = g.a0 & ~7ull;
    const uint64_t end = (g.a0 + 2ull * g.npairs + 7) & ~7ull;
    bytes = (uint32_t)(end - start) * 2;
}

// Tile t over all segments of the level.
// selc (nullable): the selection flag of segment i, cached by the caller and re-read only
// when the segment changes (a global load per tile ahead of the next tile's bulk copy
// delayed the copy)
__device__ __forceinline__ TileGeom tile_geom_all(const LevelParams& p, uint64_t t, uint32_t& i, bool* selc = nullptr) {
    const uint32_t i0 = i;
    if (i == ~0u) i = find_seg(p.tile_prefix, p.nsegs, t);
    else
        while (i + 1 < p.nsegs && p.tile_prefix[i + 1] <= t) ++i;
    const SegDesc& sd = p.segs[i];
    const uint64_t lo = sd.in_begin + (t - p.tile_prefix[i]) * (uint64_t)kTileKeys;
    TileGeom g;
    // a segment another kernel of the level handles: an empty tile (no copy, no keys)
    bool sel = true;
    if (p.seg_sel) {
        if (!selc) sel = seg_selected(p, i);
        else {
            if (i != i0) *selc = seg_selected(p, i);
            sel = *selc;
        }
    }
    g.init(p.src, lo, sel ? min(lo + kTileKeys, sd.in_begin + sd.n) : lo);
    return g;
}

template <bool IN_F64, uint32_t NBC>
__global__ void __launch_bounds__(kPNT, kPartPerSM) k_scatter(LevelParams p) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    ScatterSmem<NBC>& Q = *(ScatterSmem<NBC>*)smem_u4;
    if (p.ctrl->nan_index != ~0ull) return;
    if (p.gate && *p.gate == 0) return;
    // every child of the level is an equality fill (k_scan_children's key counters):
    // nothing moves (duplicate-heavy levels, e.g. rootdups' level 1)
    if (!p.remote && p.ctrl->keys_base + p.ctrl->keys_rec == 0) return;
    // a level partly run one-pass (seg_sel 2): only the other segments' tiles, from
    // k_kind_plan's list of every selected segment (slot 3)
    const bool lst = p.seg_sel == 2;
    const uint32_t* ks3 = p.kseg + 3 * (size_t)p.kstride;
    const uint64_t* tp3 = p.ktp + 3 * ((size_t)p.kstride + 1);
    const uint32_t nks3 = lst ? p.kplan[3].nsegs : 0u;
    const uint64_t ntl = lst ? p.kplan[3].ntiles : p.ntiles;
    auto geom = [&](uint64_t t, uint32_t& i) -> TileGeom {
        if (!lst) return tile_geom_all(p, t, i);
        if (i == ~0u) i = find_seg(tp3, nks3, t);
        else
            while (i + 1 < nks3 && tp3[i + 1] <= t) ++i;
        const SegDesc& sd = p.segs[ks3[i]];
        const uint64_t lo = sd.in_begin + (t - tp3[i]) * (uint64_t)kTileKeys;
        TileGeom g;
        g.init(p.src, lo, min(lo + kTileKeys, sd.in_begin + sd.n));
        return g;
    };
    const uint64_t per = (ntl + gridDim.x - 1) / gridDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * per;
    const uint64_t t1 = min(t0 + per, ntl);
    if (t0 >= t1) return;
    for (uint32_t b = threadIdx.x; b < NBC; b += kPNT) Q.cnt[0][b] = Q.cnt[1][b] = 0;
    TileStream TS;
    TS.init((uint8_t*)Q.tiles, Q.bars);
    // the ids ride on the keys' mbarrier: extra transaction bytes, no extra arrival
    // (added before the keys' arrive.expect_tx so the phase cannot complete early)
    auto issue_ids = [&](const TileGeom& g, int b) {
        if (threadIdx.x == 0 && g.npairs) {
            uint64_t st0;
            uint32_t bytes;
            ids_range(g, st0, bytes);
            mbar_add_tx(TS.bar + b, bytes);
            tma_load_1d(Q.sids[b], p.ids + st0, bytes, TS.bar + b);
        }
    };
    uint32_t inext = ~0u;
    TileGeom gnext = geom(t0, inext);
    issue_ids(gnext, 0);
    TS.issue(p.src, gnext, 0);
    int64_t cur = -1;
    uint64_t boff = 0;
    uint32_t nbo = 0;
    for (uint64_t tile = t0; tile < t1; ++tile) {
        const int tb = (int)((tile - t0) & 1);
        const uint32_t i = inext;
        const TileGeom g = gnext;
        uint32_t* cnt = Q.cnt[tb];
        if ((int64_t)i != cur) {
            const SegDesc& sd = p.segs[lst ? ks3[i] : i];
            boff = sd.bucket_off;
            nbo = sd.nb_max;
            cur = i;
        }
        TS.wait(g, tb);  // keys and ids of this tile have landed
        const bool al = !(g.a0 & 1);
        uint32_t idp[kPPairs];
        {
            const uint16_t* sid = Q.sids[tb] + (g.a0 & 7);
#pragma unroll
            for (int j = 0; j < kPPairs; ++j) {
                const uint32_t qq = threadIdx.x + j * kPNT;
                idp[j] = 0xffffffffu;
                if (qq < g.npairs) {
                    const uint16_t* d = sid + 2 * qq;
                    idp[j] = al ? *(const uint32_t*)d : ((uint32_t)d[0] | ((uint32_t)d[1] << 16));
                }
            }
        }
        const ulonglong2* sp = TS.buf(tb);
        uint64_t* skeys = (uint64_t*)TS.buf(tb);  // staging reuses the consumed tile buffer
        ulonglong2 v[kPPairs];
        uint32_t code[kPItems];  // bucket << 16 | rank; ~0 = not moved
#pragma unroll
        for (int j = 0; j < kPPairs; ++j) {
            uint32_t qq = threadIdx.x + j * kPNT;
            v[j] = qq < g.npairs ? sp[qq] : make_ulonglong2(0, 0);
        }
        if (IN_F64) {
#pragma unroll
            for (int j = 0; j < kPPairs; ++j) {
                v[j].x = encode(__longlong_as_double((long long)v[j].x));
                v[j].y = encode(__longlong_as_double((long long)v[j].y));
            }
        }
        // Rank within the tile. A warp whose first key slot shares one bucket
        // (sorted runs, heavy buckets) takes the warp-uniform path for the tile
        // (one atomic per warp when a slot is uniform); spread warps use plain
        // returning atomics (distinct addresses: no serialisation) without the
        // per-key uniformity votes.
        const uint32_t b00 = idp[0] & 0xffffu;
        if (__all_sync(FULL_MASK, b00 == __shfl_sync(FULL_MASK, b00, 0))) {
#pragma unroll
            for (int q = 0; q < kPItems; ++q) {
                uint32_t b = (q & 1) ? (idp[q >> 1] >> 16) : (idp[q >> 1] & 0xffffu);
                const bool ok = b != kNoMove;
                const uint32_t r = hist_rank_warp(cnt, b, ok);
                code[q] = ok ? (b << 16 | r) : 0xffffffffu;
            }
        } else {
#pragma unroll
            for (int q = 0; q < kPItems; ++q) {
                uint32_t b = (q & 1) ? (idp[q >> 1] >> 16) : (idp[q >> 1] & 0xffffu);
                const bool ok = b != kNoMove;
                code[q] = ok ? (b << 16 | atomicAdd(&cnt[b], 1u)) : 0xffffffffu;
            }
        }
        uint64_t skey = 0;
        uint32_t scode = 0xffffffffu;
        if (threadIdx.x < g.nsingle) {
            const uint64_t ix = g.single(threadIdx.x);
            uint32_t b = p.ids[ix];
            if (b != kNoMove) {
                scode = b << 16 | atomicAdd(&cnt[b], 1u);
                skey = load_key(p.src, ix, IN_F64);
            }
        }
        __syncthreads();  // (1) tile counts complete; every thread is past the previous tile
        if (tile + 1 < t1) {  // prefetch the next tile into the buffer the previous tile staged in
            gnext = geom(tile + 1, inext);
            issue_ids(gnext, tb ^ 1);
            TS.issue(p.src, gnext, tb ^ 1);
        }
        // Fused tile scan + claims at a fixed geometry: thread t owns buckets
        // [t*kPer, t*kPer + kPer) (vector load), one warp scan, warp offsets by
        // REDUX (no single-warp phase), claim atomics issued before the staging
        // and consumed after it (their latency hides behind the staging stores).
        constexpr int kPer = NBC / kPNT;
        static_assert(kPer * kPNT == NBC && (kPer == 2 || kPer == 4), "scatter geometry");
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint32_t bb = threadIdx.x * kPer;
        uint32_t cn[kPer];
        if constexpr (kPer == 2) {
            const uint2 t2 = *(const uint2*)&cnt[bb];
            cn[0] = t2.x; cn[1] = t2.y;
        } else {
            const uint4 t4 = *(const uint4*)&cnt[bb];
            cn[0] = t4.x; cn[1] = t4.y; cn[2] = t4.z; cn[3] = t4.w;
        }
        uint32_t sum = 0;
#pragma unroll
        for (int k = 0; k < kPer; ++k) sum += cn[k];
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t w = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += w;
        }
        if (lane == 31) Q.wsum[warp] = incl;
        __syncthreads();  // (2)
        const uint32_t wv = lane < kPNT / 32 ? Q.wsum[lane] : 0u;
        const uint32_t total = __reduce_add_sync(FULL_MASK, wv);
        uint32_t run = __reduce_add_sync(FULL_MASK, lane < warp ? wv : 0u) + incl - sum;
        uint32_t st[kPer];
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
            st[k] = run;
            run += cn[k];
        }
        if constexpr (kPer == 2) *(uint2*)&cnt[bb] = make_uint2(st[0], st[1]);
        else *(uint4*)&cnt[bb] = make_uint4(st[0], st[1], st[2], st[3]);
        if (threadIdx.x == 0) cnt[NBC] = total;
        __syncthreads();  // (3) tile-local bucket starts visible
        // claims strided over the threads (bucket t, t + kPNT, ...): all atomics in
        // flight while this thread stages its keys; consumed after the staging
        unsigned long long got[kPer];
        uint32_t cstart[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const uint32_t b = threadIdx.x + q * kPNT;
            got[q] = 0;
            cstart[q] = cnt[b];
            if (b < nbo) {
                const uint32_t c = cnt[b + 1] - cstart[q];
                if (c) got[q] = atomicAdd(&p.buckets[boff + b], (unsigned long long)c);
            }
        }
#pragma unroll
        for (int j = 0; j < kPItems; ++j) {
            const uint32_t c = code[j];
            if (c != 0xffffffffu) {
                const uint32_t pos = cnt[c >> 16] + (c & 0xffffu);
                skeys[pos] = (j & 1) ? v[j >> 1].y : v[j >> 1].x;
                Q.sbid[pos] = (uint16_t)(c >> 16);
            }
        }
        if (scode != 0xffffffffu) {
            const uint32_t pos = cnt[scode >> 16] + (scode & 0xffffu);
            skeys[pos] = skey;
            Q.sbid[pos] = (uint16_t)(scode >> 16);
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) Q.delta[threadIdx.x + q * kPNT] = (long long)got[q] - (long long)cstart[q];
        __syncthreads();  // (4)
#pragma unroll
        for (int q = 0; q < kTileKeys / kPNT; ++q) {  // unrolled: loads of all rows in flight
            const uint32_t j = threadIdx.x + q * kPNT;
            if (j < total) p.dst[(long long)j + Q.delta[Q.sbid[j]]] = skeys[j];
        }
        if constexpr (kPer == 2) *(uint2*)&cnt[bb] = make_uint2(0, 0);
        else *(uint4*)&cnt[bb] = make_uint4(0, 0, 0, 0);
        // staging writes (generic proxy) before the next bulk copy into this buffer,
        // which is issued after the next tile's first barrier (no end-of-tile
        // barrier: the counters alternate by tile parity)
        fence_proxy_async_smem();
    }
    // stores into peer GPUs' memory are ordered before the stream-ordered
    // barrier collective that follows this kernel (dist.cu)
    if (p.remote) __threadfence_system();
}

// ------------------------------------------------ one-pass (padded) levels
// A level whose segments all have learned models trained on samples large
// enough to predict their bucket counts does not need a histogram pass:
// classify, rank, claim and scatter in ONE pass (no k_hist pass, no stored
// bucket ids: 8 + 16 B per key instead of 10 + 18). The counts are not known
// in advance, so bucket b of a segment writes into a padded region
// [base_b, base_b + cap_b) sized from the segment's model sample (c_b of its m
// samples): cap_b = ceil(n/m (c_b + 6 sqrt(c_b) + 8)), six standard deviations
// of the sampling error. A claim past its region's end is not written and
// raises the overflow flag; the level's exact two-pass kernels (k_kind_plan /
// k_hist / k_scan_children / k_scatter, gated on Ctrl::run_exact) then run
// instead, so the result never depends on the estimate. The children are read
// at their padded offsets (SegOut::in_begin, BaseItem::src) and written at
// exact ones (SegOut::begin, BaseItem::begin): no compaction pass. The counts
// come from the root sample's bucket offsets (p.slices); the kernels take any
// number of learned segments (bucket slots at SegDesc::bucket_off).
constexpr double kDirectSigma = 6.0, kDirectSlack = 8.0;

constexpr size_t kDirectTableBytes = 20 * kDirectMaxBuckets > 2 * kRootLutCells ? 20 * kDirectMaxBuckets : 2 * kRootLutCells;

struct DirectWS {
    unsigned long long* cur;     // [slots] claim cursors (absolute positions in the padded output)
    unsigned long long* base;    // [slots] region starts
    unsigned long long* end;     // [slots] region ends
    uint32_t* ovf;               // 2: the level is not eligible, 1: a region overflowed
};
__host__ __device__ inline DirectWS direct_ws(void* w, uint64_t slots, uint32_t nsegs) {
    DirectWS d;
    d.cur = (unsigned long long*)w;
    d.base = d.cur + slots;
    d.end = d.base + slots;
    d.ovf = (uint32_t*)(d.end + slots);
    (void)nsegs;
    return d;
}
size_t direct_workspace_bytes(uint64_t slots, uint32_t nsegs) { return 8 * (3 * slots) + 16 + 0 * nsegs; }
// (ovf[0]: 2 ineligible level / alloc exceeded, 1 a region overflowed; ovf[1]: the
// one-pass level 1 left some segments to the exact kernels)
const uint32_t* direct_flag_ptr(const void* dw, uint64_t slots, uint32_t nsegs) {
    return direct_ws((void*)dw, slots, nsegs).ovf;
}

uint64_t direct_capacity_bound(uint64_t n, uint64_t m, uint32_t nb) {
    // sum_b sqrt(c_b) <= sqrt(nb m) (Cauchy-Schwarz); + 1 per bucket for the ceiling
    const double r = (double)n / (double)m;
    return (uint64_t)(r * ((double)m + kDirectSigma * sqrt((double)nb * (double)m) + kDirectSlack * nb)) + 2 * nb + 16;
}

// One CTA: the single segment's regions from the root sample's bucket offsets
// (caps, their exclusive scan, cursors) and the eligibility flag.
template <int NT>
__global__ void __launch_bounds__(NT) k_direct_setup(LevelParams p, uint64_t root_m, uint64_t alloc, DirectWS w,
                                                     double sigma, double slack) {
    griddep_wait();
    __shared__ uint64_t wsum[NT / 32 + 1];
    extern __shared__ uint64_t capv[];  // nb + 1
    const SegDesc sd = p.segs[0];
    const ModelHdr* h = (const ModelHdr*)(p.models + sd.model_off);
    const uint32_t nb = h->nbuckets;
    const bool lutm = h->kind == kRadix && (h->flags & kModelLut);  // a root cell table
    // a splitter-tree root (dup-heavy policy): regions from its first sample, if the tree
    // and its lookup table fit k_direct's table space
    const bool treem = h->kind == kTree && h->s1 >= 2 &&
                       ((tree_payload_bytes(h->leaf_origin, h->nsplit) + 15) & ~15ull) + kLutBytes <= kDirectTableBytes;
    if ((h->kind != kLearned && !lutm && !treem) || root_m == 0 || nb > kDirectMaxBuckets ||
        (h->kind == kLearned && h->B > kDirectMaxBuckets) || !p.slices) {
        if (threadIdx.x == 0) *w.ovf = 2u;  // not eligible: the exact level runs
        return;
    }
    const double r = (double)sd.n / (double)(treem ? h->s1 : root_m);
    for (uint32_t b = threadIdx.x; b < nb; b += NT) {
        const double c = (double)(p.slices[b + 1] - p.slices[b]);
        const double e = c + sigma * sqrt(c) + slack;
        capv[b] = e > 0.0 ? (uint64_t)ceil(r * e) : 0ull;
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < nb; b += NT) w.end[sd.bucket_off + b] = capv[b];
    __syncthreads();
    const uint64_t tot = block_exclusive_scan_u64<NT>(capv, nb, wsum);
    for (uint32_t b = threadIdx.x; b < nb; b += NT) {
        w.base[sd.bucket_off + b] = capv[b];
        w.cur[sd.bucket_off + b] = capv[b];
        w.end[sd.bucket_off + b] += capv[b];
    }
    if (threadIdx.x == 0) *w.ovf = tot > alloc ? 2u : 0u;  // (the host's bound holds)
}

struct DirectSmem {
    uint64_t bars[2];
    ulonglong2 tiles[2][kTileKeys / 2];  // TMA tile buffers; the consumed one stages the tile
    long long delta[kDirectMaxBuckets];  // per bucket: claimed position - tile-local start
    alignas(16) uint32_t cnt[2][kDirectMaxBuckets + 4];
    uint16_t sbid[kTileKeys];
    uint32_t wsum[kPNT / 32 + 1];
    // the segment model's compiled table, cell table, or splitter tree + its lookup table (kstate_load)
    alignas(16) uint8_t table[kDirectTableBytes];
    uint8_t iseq[kDirectMaxBuckets];  // tree roots: equality buckets (their keys are counted, not moved)
};

static_assert(sizeof(DirectSmem) + 1024 <= 233472 / kPartPerSM, "one-pass level: kPartPerSM CTAs per SM");

// One segment (level 0), its model table loaded once. MODE: the root's
// classifier -- 0 RMI, 1 linear cell table, 2 binade (log) cell table. The
// host launches all three; the ones that do not match the model built on the
// device return at once (one kernel with all three classifiers spilled).
template <int MODE>
__device__ __forceinline__ uint32_t direct_classify(const KState& S, uint64_t x) {
    // (MODE 4: the one-pass level 1 -- every segment a linear cell table, see launch_direct_multi)
    if constexpr (MODE == 0) return kclassify<kLearned>(S, x);
    else if constexpr (MODE == 3) return kclassify<kTree>(S, x) & 0x7fffffffu;
    else if constexpr (MODE == 2) return S.rlut[binade_cell(x, S.rtab, (uint32_t)S.rmin, S.rtabn, S.rcells)];
    else {
        if (S.shift >= 32) {
            const uint32_t h = (uint32_t)(x >> 32) >> (S.shift - 32);
            return S.rlut[h > S.rorg ? min(h - S.rorg, S.rcells - 1) : 0u];
        }
        return S.rlut[lut_cell(x, S.rmin, S.shift, S.rcells)];
    }
}
template <bool IN_F64, int MODE>
__global__ void __launch_bounds__(kPNT, kPartPerSM) k_direct(LevelParams p, DirectWS w) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    DirectSmem& Q = *(DirectSmem*)smem_u4;
    constexpr uint32_t NBC = kDirectMaxBuckets;
    if (*w.ovf || p.ctrl->nan_index != ~0ull) return;
    if (MODE != 4) {
        const ModelHdr* h0 = (const ModelHdr*)(p.models + p.segs[0].model_off);
        const int mode = h0->kind == kRadix ? ((h0->flags & kModelLog) ? 2 : 1) : (h0->kind == kTree ? 3 : 0);
        if (mode != MODE) return;
    }
    const uint64_t per = (p.ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t0 = (uint64_t)blockIdx.x * per;
    const uint64_t t1 = min(t0 + per, p.ntiles);
    if (t0 >= t1) return;
    for (uint32_t b = threadIdx.x; b < NBC; b += kPNT) Q.cnt[0][b] = Q.cnt[1][b] = 0;
    TileStream TS;
    TS.init((uint8_t*)Q.tiles, Q.bars);
    uint32_t inext = ~0u;
    bool selc = true;
    TileGeom gnext = tile_geom_all(p, t0, inext, &selc);
    TS.issue(p.src, gnext, 0);
    KState S;
    if constexpr (MODE == 3) {  // splitter tree + its lookup table; equality buckets flagged
        __shared__ uint32_t lut_red;
        const ModelHdr* th = (const ModelHdr*)(p.models + p.segs[0].model_off);
        const size_t tb = (tree_payload_bytes(th->leaf_origin, th->nsplit) + 15) & ~15ull;
        kstate_load<kTree>(S, p.models + p.segs[0].model_off, Q.table, (uint16_t*)(Q.table + tb), &lut_red);
        for (uint32_t b = threadIdx.x; b < kDirectMaxBuckets; b += kPNT) Q.iseq[b] = 0;
        __syncthreads();
        for (uint32_t i = threadIdx.x; i < S.nsplit; i += kPNT)
            if (S.eqo[i + 1] - S.eqo[i] > 1) Q.iseq[S.eqo[i] + 1] = 1;
        __syncthreads();
    } else if constexpr (MODE == 0) {
        kstate_load<kLearned>(S, p.models + p.segs[0].model_off, Q.table);
    } else if constexpr (MODE != 4) {
        kstate_load<kRadix>(S, p.models + p.segs[0].model_off, Q.table);
    }
    if constexpr (MODE == 4) {
        // no table yet: a CTA whose first segments belong to the exact kernels classifies
        // its empty tiles' zero slots unconditionally -- through a valid (unused) table
        S.nb = 0; S.rmin = 0; S.shift = 0; S.fill = false; S.rcells = 1; S.rorg = 0;
        S.rtab = nullptr; S.rtabn = 0;
        S.rlut = (const uint16_t*)Q.table;
    }
    uint64_t boff = p.segs[0].bucket_off;
    uint32_t nb = MODE == 4 ? 0u : S.nb;
    uint32_t curseg = ~0u;
    bool ovf = false;
    for (uint64_t tile = t0; tile < t1; ++tile) {
        const int tb = (int)((tile - t0) & 1);
        const TileGeom g = gnext;
        uint32_t* cnt = Q.cnt[tb];
        if constexpr (MODE == 4) {  // (CTA-uniform) the tile's segment's table into shared memory
            // (a segment the exact kernels take has another model kind -- a tree, an
            // RMI: its tiles are empty and its header is not read as a cell table)
            const uint32_t si = inext;
            if (si != curseg) {
                curseg = si;
                nb = 0;
                if (selc) {
                    kstate_load<kRadix>(S, p.models + p.segs[si].model_off, Q.table);
                    boff = p.segs[si].bucket_off;
                    nb = S.nb;
                }
            }
        }
        TS.wait(g, tb);
        const ulonglong2* sp = TS.buf(tb);
        uint64_t* skeys = (uint64_t*)TS.buf(tb);  // staging reuses the consumed tile buffer
        ulonglong2 v[kPPairs];
#pragma unroll
        for (int j = 0; j < kPPairs; ++j) {
            const uint32_t qq = threadIdx.x + j * kPNT;
            v[j] = qq < g.npairs ? sp[qq] : make_ulonglong2(0, 0);
        }
        if (IN_F64) {
            bool anynan = false;
#pragma unroll
            for (int j = 0; j < kPPairs; ++j)
                anynan |= (threadIdx.x + j * kPNT < g.npairs) &&
                          (isnan(__longlong_as_double((long long)v[j].x)) | isnan(__longlong_as_double((long long)v[j].y)));
            if (anynan) {
#pragma unroll
                for (int j = 0; j < kPPairs; ++j) {
                    const uint32_t q = threadIdx.x + j * kPNT;
                    if (q < g.npairs) {
                        if (isnan(__longlong_as_double((long long)v[j].x)))
                            atomicMin(&p.ctrl->nan_index, (unsigned long long)(g.a0 + 2 * q));
                        if (isnan(__longlong_as_double((long long)v[j].y)))
                            atomicMin(&p.ctrl->nan_index, (unsigned long long)(g.a0 + 2 * q + 1));
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < kPPairs; ++j) {
                v[j].x = encode(__longlong_as_double((long long)v[j].x));
                v[j].y = encode(__longlong_as_double((long long)v[j].y));
            }
        }
        uint32_t code[kPItems];  // bucket << 16 | rank within the tile; ~0 = no key
        {
            uint32_t bk[kPItems];
            if constexpr (MODE == 0) {
                classify16<kLearned>(S, v, bk);
            } else if constexpr (MODE == 3) {
                classify16<kTree>(S, v, bk);
#pragma unroll
                for (int q = 0; q < kPItems; ++q) bk[q] &= 0x7fffffffu;
            } else {
#pragma unroll
                for (int q = 0; q < kPItems; ++q) bk[q] = direct_classify<MODE>(S, (q & 1) ? v[q >> 1].y : v[q >> 1].x);
            }
#pragma unroll
            for (int q = 0; q < kPItems; ++q) {
                const bool ok = threadIdx.x + (q >> 1) * kPNT < g.npairs;
                const uint32_t b = ok ? bk[q] : 0u;
                code[q] = ok ? (b << 16 | atomicAdd(&cnt[b], 1u)) : 0xffffffffu;
            }
        }
        uint64_t skey = 0;
        uint32_t scode = 0xffffffffu;
        if (threadIdx.x < g.nsingle) {
            const uint64_t ix = g.single(threadIdx.x);
            uint64_t k = ((const uint64_t*)p.src)[ix];
            if (IN_F64) {
                const double d = __longlong_as_double((long long)k);
                if (isnan(d)) atomicMin(&p.ctrl->nan_index, (unsigned long long)ix);
                k = encode(d);
            }
            const uint32_t b = direct_classify<MODE>(S, k);
            scode = b << 16 | atomicAdd(&cnt[b], 1u);
            skey = k;
        }
        __syncthreads();  // (1) tile counts complete; every thread is past the previous tile
        if (tile + 1 < t1) {
            gnext = tile_geom_all(p, tile + 1, inext, &selc);
            TS.issue(p.src, gnext, tb ^ 1);
        }
        constexpr int kPer = NBC / kPNT;
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        const uint32_t bb = threadIdx.x * kPer;
        const uint2 t2 = *(const uint2*)&cnt[bb];
        const uint32_t cn0 = t2.x, cn1 = t2.y, sum = cn0 + cn1;
        uint32_t incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t x = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += x;
        }
        if (lane == 31) Q.wsum[warp] = incl;
        __syncthreads();  // (2)
        const uint32_t wv = lane < kPNT / 32 ? Q.wsum[lane] : 0u;
        const uint32_t total = __reduce_add_sync(FULL_MASK, wv);
        const uint32_t run = __reduce_add_sync(FULL_MASK, lane < warp ? wv : 0u) + incl - sum;
        *(uint2*)&cnt[bb] = make_uint2(run, run + cn0);
        if (threadIdx.x == 0) cnt[NBC] = total;
        __syncthreads();  // (3) tile-local bucket starts visible
        // claims (all in flight while this thread stages its keys), the region
        // ends loaded beside them; both consumed after the staging
        unsigned long long got[kPer], lim[kPer];
        uint32_t cstart[kPer], ccnt[kPer];
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const uint32_t b = threadIdx.x + q * kPNT;
            got[q] = 0;
            lim[q] = ~0ull;
            cstart[q] = cnt[b];
            ccnt[q] = 0;
            if (b < nb) {
                ccnt[q] = cnt[b + 1] - cstart[q];
                if (ccnt[q]) {
                    got[q] = atomicAdd(&w.cur[boff + b], (unsigned long long)ccnt[q]);
                    lim[q] = w.end[boff + b];
                }
            }
        }
#pragma unroll
        for (int j = 0; j < kPItems; ++j) {
            const uint32_t c = code[j];
            if (c != 0xffffffffu) {
                const uint32_t pos = cnt[c >> 16] + (c & 0xffffu);
                skeys[pos] = (j & 1) ? v[j >> 1].y : v[j >> 1].x;
                Q.sbid[pos] = (uint16_t)(c >> 16);
            }
        }
        if (scode != 0xffffffffu) {
            const uint32_t pos = cnt[scode >> 16] + (scode & 0xffffu);
            skeys[pos] = skey;
            Q.sbid[pos] = (uint16_t)(scode >> 16);
        }
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const bool full = ccnt[q] && got[q] + ccnt[q] > lim[q];  // region full: nothing of this run is written
            ovf |= full;
            // (tree roots: an equality bucket's keys are counted by its claims, filled later)
            const bool skip = full || (MODE == 3 && Q.iseq[threadIdx.x + q * kPNT]);
            Q.delta[threadIdx.x + q * kPNT] = skip ? LLONG_MIN : (long long)got[q] - (long long)cstart[q];
        }
        __syncthreads();  // (4)
#pragma unroll
        for (int q = 0; q < kTileKeys / kPNT; ++q) {
            const uint32_t j = threadIdx.x + q * kPNT;
            if (j < total) {
                const long long d = Q.delta[Q.sbid[j]];
                if (d != LLONG_MIN) p.dst[(long long)j + d] = skeys[j];
            }
        }
        *(uint2*)&cnt[bb] = make_uint2(0, 0);
        fence_proxy_async_smem();
    }
    if (ovf) atomicOr(w.ovf, 1u);
}

// One CTA per segment: unless the level is ineligible or a region overflowed,
// every non-empty bucket becomes a next-level segment, read at its padded base
// (SegOut::in_begin) and written at its exact offset (exclusive scan of the
// counts) -- small ones too: a base-case item reads where it writes, and the
// one-pass level only runs with >= 64 Ki keys per bucket on average. Otherwise
// the exact two-pass level runs (Ctrl::run_exact).
template <int NT>
__global__ void __launch_bounds__(NT) k_direct_children(LevelParams p, DirectWS w, int64_t base_delta) {
    griddep_wait();
    __shared__ uint64_t wsum[NT / 32 + 1];
    __shared__ uint32_t lbase;
    __shared__ uint32_t lcount[4], gbase[4];
    __shared__ unsigned long long lkeys, lfill;
    __shared__ uint8_t iseqs[kDirectMaxBuckets];
    __shared__ uint64_t eqvs[kDirectMaxBuckets];
    extern __shared__ uint64_t cntv[];  // nb + 1
    if (p.ctrl->nan_index != ~0ull) return;
    if (*w.ovf) {
        if (blockIdx.x == 0 && threadIdx.x == 0) { p.ctrl->direct = 0; p.ctrl->run_exact = 1; }
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { p.ctrl->direct = 1; p.ctrl->run_exact = 0; }
    const SegDesc sd = p.segs[blockIdx.x];
    const uint32_t nb = ((const ModelHdr*)(p.models + sd.model_off))->nbuckets;
    for (uint32_t b = threadIdx.x; b < nb; b += NT) cntv[b] = w.cur[sd.bucket_off + b] - w.base[sd.bucket_off + b];
    __syncthreads();
    block_exclusive_scan_u64<NT>(cntv, nb, wsum);
    if (threadIdx.x == 0) { lbase = 0; lkeys = 0; lfill = 0; }
    if (threadIdx.x < 4) lcount[threadIdx.x] = 0;
    const ModelHdr* mh = (const ModelHdr*)(p.models + sd.model_off);
    const bool tree = mh->kind == kTree;  // (its equality buckets become fills; its offsets index the first sample)
    for (uint32_t b = threadIdx.x; b < kDirectMaxBuckets; b += NT) iseqs[b] = 0;
    __syncthreads();
    if (tree) {
        const MView m = model_view(p.models + sd.model_off);
        for (uint32_t i = threadIdx.x; i < mh->nsplit; i += NT)
            if (m.eqo[i + 1] - m.eqo[i] > 1) {
                iseqs[m.eqo[i] + 1] = 1;
                eqvs[m.eqo[i] + 1] = m.spl[i];
            }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // children of at most the base-case capacity go straight to the base cases
    // (read at the padded base through base_delta: BaseItem::rd is relative to
    // the base kernels' source pointer), the rest become level-1 segments
    for (uint32_t b0 = 0; b0 < nb; b0 += NT) {  // CTA-uniform rounds
        const uint32_t b = b0 + threadIdx.x;
        uint64_t st = 0, len = 0;
        if (b < nb) {
            st = cntv[b];
            len = (b + 1 < nb ? cntv[b + 1] : sd.n) - st;
        }
        const int cls = len == 0 ? -1
                        : (tree && iseqs[b]) ? 4
                        : (len <= p.base_cap[2] ? (len <= p.base_cap[0] ? 0 : (len <= p.base_cap[1] ? 1 : 2)) : 3);
        const unsigned m = __ballot_sync(FULL_MASK, cls == 3);
        uint32_t wb = 0;
        if (lane == 0 && m) wb = atomicAdd(&lbase, (uint32_t)__popc(m));
        wb = __shfl_sync(FULL_MASK, wb, 0);
        uint32_t li = 0;
#pragma unroll
        for (int c = 0; c < 5; ++c) {
            if (c == 3) continue;  // (recursion: lbase above)
            const unsigned mc = __ballot_sync(FULL_MASK, cls == c);
            if (mc) {
                const int leader = __ffs(mc) - 1;
                const int slot = c == 4 ? 3 : c;
                uint32_t base = 0;
                if (lane == leader) base = atomicAdd(&lcount[slot], (uint32_t)__popc(mc));
                base = __shfl_sync(FULL_MASK, base, leader);
                if (cls == c) li = base + __popc(mc & lt);
            }
        }
        unsigned long long kb = (cls >= 0 && cls < 3) ? (unsigned long long)len : 0ull;
        unsigned long long kf = cls == 4 ? (unsigned long long)len : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            kb += __shfl_xor_sync(FULL_MASK, kb, o);
            kf += __shfl_xor_sync(FULL_MASK, kf, o);
        }
        if (lane == 0 && kb) atomicAdd(&lkeys, kb);
        if (lane == 0 && kf) atomicAdd(&lfill, kf);
        __syncthreads();
        if (threadIdx.x < 4) {
            const uint32_t c = lcount[threadIdx.x];
            unsigned int* ctr = threadIdx.x == 3 ? &p.ctrl->n_fill : &p.ctrl->n_base[threadIdx.x];
            gbase[threadIdx.x] = c ? atomicAdd(ctr, c) : 0u;
            lcount[threadIdx.x] = 0;
        }
        __syncthreads();
        if (cls == 3) {
            const uint32_t e0 = wb + __popc(m & lt);
            uint64_t ps = 0;
            if (p.slices && !tree) {
                const uint32_t o = p.slices[b], l = p.slices[b + 1] - o;
                if (l >= kMinSlice) ps = (uint64_t)o << 24 | min(l, 0xffffffu);
            }
            const uint32_t depth = sd.depth + 1;
            const uint32_t flags = (len == sd.n || depth > p.depth_cap) ? kSegForceRadix : 0u;
            const uint32_t e = p.ctrl->n_rec + e0;  // (one segment: the list starts empty)
            if (e < p.list_cap) p.rec[e] = SegOut{sd.begin + st, len, depth, flags, ps, w.base[sd.bucket_off + b]};
            else atomicOr(&p.ctrl->err, 4u);
        } else if (cls == 4) {  // equality bucket: every key equals the splitter
            const uint32_t e = gbase[3] + li;
            if (e < p.list_cap) p.fill[e] = FillItem{sd.begin + st, len, eqvs[b], 0};
            else atomicOr(&p.ctrl->err, 1u);
        } else if (cls >= 0) {
            const uint32_t e = gbase[cls] + li;
            if (e < p.list_cap)
                p.base[cls][e] = BaseItem{sd.begin + st, len, base_delta + (int64_t)w.base[sd.bucket_off + b]};
            else atomicOr(&p.ctrl->err, 2u);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        p.ctrl->n_rec += lbase;
        p.ctrl->keys_base += lkeys;
        p.ctrl->keys_fill += lfill;
        p.ctrl->keys_rec += sd.n - lkeys - lfill;
    }
}

// ------------------------------------------------ one-pass level 1 (multi)
// Every segment of a level >= 1 with a linear cell table and a slice of the
// parent's sorted sample: bucket b of segment s gets a padded region sized from
// its slice count (k_mdirect_caps), regions laid out segment after segment
// (k_mdirect_scan, k_mdirect_bases), one pass classifies / ranks / claims /
// scatters all tiles (k_direct<false, 4>), and k_mdirect_children lists the
// children (base cases read at their padded base). Any ineligible segment or
// overflowing region runs the exact two-pass level instead (Ctrl::run_exact).
__global__ void __launch_bounds__(256) k_mdirect_caps(LevelParams p, DirectWS w, const uint64_t* psample,
                                                      uint64_t* seg_tot, double sigma, double slack, uint32_t* segd) {
    griddep_wait();
    __shared__ uint32_t hist[kDirectMaxBuckets];
    __shared__ uint64_t red[256 / 32];
    const SegDesc sd = p.segs[blockIdx.x];
    const ModelHdr* h = (const ModelHdr*)(p.models + sd.model_off);
    const uint32_t len = (uint32_t)(sd.pslice & 0xffffffu);
    const bool ok = psample && h->kind == kRadix && (h->flags & kModelLut) && !(h->flags & kModelLog) &&
                    h->nbuckets <= kDirectMaxBuckets && len >= 2 && !(sd.flags & kSegForceRadix);
    if (!ok) {  // another model kind: the exact two-pass kernels take this segment
        if (threadIdx.x == 0) { segd[blockIdx.x] = 0; seg_tot[blockIdx.x] = 0; atomicOr(w.ovf + 1, 1u); }
        return;
    }
    if (threadIdx.x == 0) segd[blockIdx.x] = 1;
    const uint32_t nb = h->nbuckets;
    for (uint32_t b = threadIdx.x; b < nb; b += 256) hist[b] = 0;
    __syncthreads();
    const uint16_t* lut = (const uint16_t*)(h + 1);
    const uint64_t* smp = psample + (sd.pslice >> 24);
    for (uint32_t i = threadIdx.x; i < len; i += 256)
        atomicAdd(&hist[lut[lut_cell(smp[i], h->radix_min, h->shift, h->B)]], 1u);
    __syncthreads();
    const double r = (double)sd.n / (double)len;
    uint64_t tot = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += 256) {
        const double c = (double)hist[b];
        const double e = c + sigma * sqrt(c) + slack;
        const uint64_t cap = e > 0.0 ? (uint64_t)ceil(r * e) : 0ull;
        w.end[sd.bucket_off + b] = cap;
        tot += cap;
    }
    tot = block_reduce_sum_u64<256>(tot, red);
    if (threadIdx.x == 0) seg_tot[blockIdx.x] = tot;
}
__global__ void __launch_bounds__(1024) k_mdirect_scan(uint32_t nsegs, uint64_t* seg_tot, uint64_t alloc, DirectWS w) {
    griddep_wait();
    __shared__ uint64_t wsum[1024 / 32 + 1];
    if (*w.ovf) return;
    const uint64_t tot = block_exclusive_scan_u64<1024>(seg_tot, nsegs, wsum);
    if (threadIdx.x == 0 && tot > alloc) *w.ovf = 2u;
}
__global__ void __launch_bounds__(256) k_mdirect_bases(LevelParams p, DirectWS w, const uint64_t* seg_base) {
    griddep_wait();
    __shared__ uint64_t capv[kDirectMaxBuckets];
    __shared__ uint64_t wsum[256 / 32 + 1];
    if (*w.ovf || !p.seg_direct[blockIdx.x]) return;
    const SegDesc sd = p.segs[blockIdx.x];
    const uint32_t nb = ((const ModelHdr*)(p.models + sd.model_off))->nbuckets;
    for (uint32_t b = threadIdx.x; b < nb; b += 256) capv[b] = w.end[sd.bucket_off + b];
    __syncthreads();
    block_exclusive_scan_u64<256>(capv, nb, wsum);
    const uint64_t s0 = seg_base[blockIdx.x];
    for (uint32_t b = threadIdx.x; b < nb; b += 256) {
        const uint64_t c = w.end[sd.bucket_off + b];
        w.base[sd.bucket_off + b] = s0 + capv[b];
        w.cur[sd.bucket_off + b] = s0 + capv[b];
        w.end[sd.bucket_off + b] = s0 + capv[b] + c;
    }
}
template <int NT>
__global__ void __launch_bounds__(NT) k_mdirect_children(LevelParams p, DirectWS w, int64_t base_delta) {
    griddep_wait();
    __shared__ uint64_t wsum[NT / 32 + 1];
    __shared__ uint32_t lcount[4], gbase[4];
    __shared__ unsigned long long lkeys[2];  // base, rec
    __shared__ uint64_t cntv[kDirectMaxBuckets];
    if (p.ctrl->nan_index != ~0ull) return;
    if (*w.ovf) {  // a region overflowed: the exact two-pass level takes every segment
        if (threadIdx.x == 0) const_cast<uint32_t*>(p.seg_direct)[blockIdx.x] = 0;
        if (blockIdx.x == 0 && threadIdx.x == 0) { p.ctrl->direct = 0; p.ctrl->run_exact = 1; }
        return;
    }
    // (some segments of another model kind: the exact kernels run for those)
    if (blockIdx.x == 0 && threadIdx.x == 0) { p.ctrl->direct = 1; p.ctrl->run_exact = w.ovf[1] ? 1u : 0u; }
    if (!p.seg_direct[blockIdx.x]) return;
    const SegDesc sd = p.segs[blockIdx.x];
    const uint32_t nb = ((const ModelHdr*)(p.models + sd.model_off))->nbuckets;
    for (uint32_t b = threadIdx.x; b < nb; b += NT) cntv[b] = w.cur[sd.bucket_off + b] - w.base[sd.bucket_off + b];
    if (threadIdx.x < 4) lcount[threadIdx.x] = 0;
    if (threadIdx.x < 2) lkeys[threadIdx.x] = 0;
    __syncthreads();
    block_exclusive_scan_u64<NT>(cntv, nb, wsum);
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t b0 = 0; b0 < nb; b0 += NT) {  // CTA-uniform rounds
        const uint32_t b = b0 + threadIdx.x;
        uint64_t st = 0, len = 0;
        if (b < nb) {
            st = cntv[b];
            len = (b + 1 < nb ? cntv[b + 1] : sd.n) - st;
        }
        const int cls = len == 0 ? -1 : (len <= p.base_cap[2] ? (len <= p.base_cap[0] ? 0 : (len <= p.base_cap[1] ? 1 : 2)) : 3);
        uint32_t li = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const unsigned mc = __ballot_sync(FULL_MASK, cls == c);
            if (mc) {
                const int leader = __ffs(mc) - 1;
                uint32_t base = 0;
                if (lane == leader) base = atomicAdd(&lcount[c], (uint32_t)__popc(mc));
                base = __shfl_sync(FULL_MASK, base, leader);
                if (cls == c) li = base + __popc(mc & lt);
            }
        }
        unsigned long long kb = (cls >= 0 && cls < 3) ? (unsigned long long)len : 0ull;
        unsigned long long kr = cls == 3 ? (unsigned long long)len : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            kb += __shfl_xor_sync(FULL_MASK, kb, o);
            kr += __shfl_xor_sync(FULL_MASK, kr, o);
        }
        if (lane == 0 && kb) atomicAdd(&lkeys[0], kb);
        if (lane == 0 && kr) atomicAdd(&lkeys[1], kr);
        __syncthreads();
        if (threadIdx.x < 4) {
            const uint32_t c = lcount[threadIdx.x];
            unsigned int* ctr = threadIdx.x == 3 ? &p.ctrl->n_rec : &p.ctrl->n_base[threadIdx.x];
            gbase[threadIdx.x] = c ? atomicAdd(ctr, c) : 0u;
            lcount[threadIdx.x] = 0;
        }
        __syncthreads();
        if (cls == 3) {
            const uint32_t e = gbase[3] + li;
            const uint32_t depth = sd.depth + 1;
            const uint32_t flags = (len == sd.n || depth > p.depth_cap) ? kSegForceRadix : 0u;
            if (e < p.list_cap) p.rec[e] = SegOut{sd.begin + st, len, depth, flags, 0ull, w.base[sd.bucket_off + b]};
            else atomicOr(&p.ctrl->err, 4u);
        } else if (cls >= 0) {
            const uint32_t e = gbase[cls] + li;
            if (e < p.list_cap)
                p.base[cls][e] = BaseItem{sd.begin + st, len, base_delta + (int64_t)w.base[sd.bucket_off + b]};
            else atomicOr(&p.ctrl->err, 2u);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        if (lkeys[0]) atomicAdd(&p.ctrl->keys_base, lkeys[0]);
        if (lkeys[1]) atomicAdd(&p.ctrl->keys_rec, lkeys[1]);
    }
}

size_t direct_multi_workspace_bytes(uint64_t slots, uint32_t nsegs) {
    return direct_workspace_bytes(slots, nsegs) + 16 * (size_t)nsegs + 64;
}
// the per-segment one-pass flags live in the caller's seg_direct array (LevelParams)

void launch_direct_multi(const LevelParams& p, const uint64_t* psample, uint64_t alloc_keys, void* dw, uint64_t slots,
                         int grid, cudaStream_t st, bool test_overflow, const uint64_t* base_src) {
    const DirectWS w = direct_ws(dw, slots, p.nsegs);
    uint64_t* seg_tot = (uint64_t*)((uint8_t*)dw + ((direct_workspace_bytes(slots, p.nsegs) + 15) & ~(size_t)15));
    const double sigma = test_overflow ? -kDirectSigma : kDirectSigma, slack = test_overflow ? 0.0 : kDirectSlack;
    cudaMemsetAsync(w.ovf, 0, 8, st);
    pdl(k_mdirect_caps, p.nsegs, 256, 0, st, p, w, psample, seg_tot, sigma, slack, (uint32_t*)p.seg_direct);
    pdl(k_mdirect_scan, 1, 1024, 0, st, p.nsegs, seg_tot, alloc_keys, w);
    pdl(k_mdirect_bases, p.nsegs, 256, 0, st, p, w, (const uint64_t*)seg_tot);
    constexpr size_t sm = sizeof(DirectSmem);
    pdl(k_direct<false, 4>, grid, kPNT, sm, st, p, w);
    pdl(k_mdirect_children<1024>, p.nsegs, 1024, 0, st, p, w, (int64_t)(p.dst - base_src));
}

void launch_direct(const LevelParams& p, int in_f64, uint64_t root_m, uint64_t alloc_keys, void* dw, uint64_t slots,
                   int grid, cudaStream_t st, bool test_overflow, const uint64_t* base_src) {
    const DirectWS w = direct_ws(dw, slots, p.nsegs);
    const double sigma = test_overflow ? -kDirectSigma : kDirectSigma, slack = test_overflow ? 0.0 : kDirectSlack;
    const size_t cap_sm = 8 * ((size_t)kDirectMaxBuckets + 2);
    pdl(k_direct_setup<1024>, 1, 1024, cap_sm, st, p, root_m, alloc_keys, w, sigma, slack);
    constexpr size_t sm = sizeof(DirectSmem);
    if (in_f64) {
        pdl(k_direct<true, 1>, grid, kPNT, sm, st, p, w);
        pdl(k_direct<true, 2>, grid, kPNT, sm, st, p, w);
        pdl(k_direct<true, 0>, grid, kPNT, sm, st, p, w);
        pdl(k_direct<true, 3>, grid, kPNT, sm, st, p, w);
    } else {
        pdl(k_direct<false, 1>, grid, kPNT, sm, st, p, w);
        pdl(k_direct<false, 2>, grid, kPNT, sm, st, p, w);
        pdl(k_direct<false, 0>, grid, kPNT, sm, st, p, w);
        pdl(k_direct<false, 3>, grid, kPNT, sm, st, p, w);
    }
    pdl(k_direct_children<1024>, p.nsegs, 1024, cap_sm, st, p, w, (int64_t)(p.dst - base_src));
}

// ------------------------------------------------------------- launchers
static const uint32_t kTreeCap = (uint32_t)(kTreeCapBytes + kLutBytes);

void partition_init(int optin) {
    allow_smem(k_hist<true, kLearned>, optin);
    allow_smem(k_hist<false, kLearned>, optin);
    allow_smem(k_hist<true, kTree>, optin);
    allow_smem(k_hist<false, kTree>, optin);
    allow_smem(k_hist<true, kRadix>, optin);
    allow_smem(k_hist<false, kRadix>, optin);
    allow_smem(k_scatter<true, 1024>, optin);
    allow_smem(k_scatter<false, 1024>, optin);
    allow_smem(k_scatter<true, kMaxNB>, optin);
    allow_smem(k_scatter<false, kMaxNB>, optin);
    allow_smem(k_direct<true, 0>, optin);
    allow_smem(k_direct<false, 0>, optin);
    allow_smem(k_direct<true, 1>, optin);
    allow_smem(k_direct<false, 1>, optin);
    allow_smem(k_direct<true, 2>, optin);
    allow_smem(k_direct<false, 2>, optin);
    allow_smem(k_direct<true, 3>, optin);
    allow_smem(k_direct<false, 3>, optin);
    allow_smem(k_direct<false, 4>, optin);
    allow_smem(k_direct_setup<1024>, optin);
    allow_smem(k_direct_children<1024>, optin);
    allow_smem(k_scan_children<128>, optin);
    allow_smem(k_scan_children<512>, optin);
    allow_smem(k_scan_children<1024>, optin);
}

void launch_kind_plan(const LevelParams& p, cudaStream_t st) {
    pdl(k_kind_plan, 1, kPlanNT, 0, st, p);
}

void launch_hist(const LevelParams& p, int in_f64, uint32_t kinds, uint32_t max_rmi_b, int grid, cudaStream_t st) {
    const size_t table_bytes = 20 * (size_t)max_rmi_b;
    size_t sm_r = 16 + 4 * (size_t)kMaxNB + 2 * kTileBytes, sm_t = sm_r + kTreeCap, sm_l = sm_r + table_bytes;
    sm_r += 2 * (size_t)(kLutModelMaxCells > kRootLutCells ? kLutModelMaxCells : kRootLutCells);  // (radix kind: a cell table)
    if (kinds & 1) {
        const int gl = grid;
        if (in_f64) pdl(k_hist<true, kLearned>, gl, kPNT, sm_l, st, p);
        else pdl(k_hist<false, kLearned>, gl, kPNT, sm_l, st, p);
    }
    if (kinds & 2) {  // tree payload in shared memory: two CTAs per SM
        const int gt = grid;
        if (in_f64) pdl(k_hist<true, kTree>, gt, kPNT, sm_t, st, p);
        else pdl(k_hist<false, kTree>, gt, kPNT, sm_t, st, p);
    }
    if (kinds & 4) {
        if (in_f64) pdl(k_hist<true, kRadix>, grid, kPNT, sm_r, st, p);
        else pdl(k_hist<false, kRadix>, grid, kPNT, sm_r, st, p);
    }
}

void launch_scan_children(const LevelParams& p, uint32_t max_nb, cudaStream_t st) {
    if (!p.nsegs) return;
    const size_t sm = 17 * (size_t)max_nb + 16;  // cnt + eqval (u64) + iseq (u8) per bucket slot
    if (max_nb <= 256) pdl(k_scan_children<128>, p.nsegs, 128, sm, st, p);
    else if (max_nb <= 512) pdl(k_scan_children<512>, p.nsegs, 512, sm, st, p);
    else pdl(k_scan_children<1024>, p.nsegs, 1024, sm, st, p);
}

void launch_scatter(const LevelParams& p, int in_f64, uint32_t nb_cap, int grid, cudaStream_t st) {
    if (nb_cap <= 1024) {
        constexpr size_t sm = sizeof(ScatterSmem<1024>);
        if (in_f64) pdl(k_scatter<true, 1024>, grid, kPNT, sm, st, p);
        else pdl(k_scatter<false, 1024>, grid, kPNT, sm, st, p);
    } else {
        constexpr size_t sm = sizeof(ScatterSmem<kMaxNB>);
        if (in_f64) pdl(k_scatter<true, kMaxNB>, grid, kPNT, sm, st, p);
        else pdl(k_scatter<false, kMaxNB>, grid, kPNT, sm, st, p);
    }
}

}  // namespace lsort_dev
