// models.cu -- partition-model construction on the device (Alg. 5,
// SPEC.md:375-383).
//
//   k_build_models   one CTA per segment: device-drawn samples (Rng stream of
//                    the segment, rng.hpp:35-37), shared-memory sample sort,
//                    duplicate fraction (models.cpp:187-193), then RMI
//                    training (models.cpp:14-131) or SplitterTree::build
//                    (models.cpp:133-185) for samples <= 16384 keys.
//   k_first_sample   the same policy step for a big segment (first sample only).
//   k_gather         device-wide gather of a big RMI sample.
//   k_train_*        multi-CTA RMI training over a sorted sample in global
//                    memory: deterministic chunked root sums, per-submodel
//                    fits (sequential = bit-exact for slices <= 512 samples,
//                    one CTA per larger slice), single-CTA monotone clamps.
#include <algorithm>

#include "kernels_common.cuh"
#include "smemsort.cuh"

namespace lsort_dev {

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
__device__ __noinline__ void train_rmi_block(const uint64_t* s, uint32_t n, uint32_t B, ModelHdr* hdr, RmiEntry* E,
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
    compile_learned((uint8_t*)hdr, threadIdx.x, NT);
    __syncthreads();
}

// SplitterTree::build (models.cpp:133-185) by one CTA from a sorted sample in
// shared memory. Scratch: u32[2k].
template <int NT>
__device__ __noinline__ void tree_build_block(const uint64_t* s, uint32_t n, uint32_t k, bool eq_mode, ModelHdr* hdr,
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

// Model-building CTA configurations: NT threads, sample capacity CAP. The
// sample is sorted in shared memory by SmemSort (rolled loops: the former
// register-array sorter made this kernel 52K SASS instructions and
// instruction-fetch bound).
template <int NT, int CAP>
struct ModelCfg {
    static constexpr int kCap = CAP;
    using SS = SmemSort<NT, CAP, CAP / 2>;
    struct Smem {
        typename SS::Smem sort;  // sort.A holds the sorted sample
        union {
            struct {
                uint32_t first[LSORT_MAX_RMI_DEV + 1];
                double lo[LSORT_MAX_RMI_DEV];
                double hi[LSORT_MAX_RMI_DEV];
                uint32_t big[LSORT_MAX_RMI_DEV];
                double red[2 * (NT / 32)];
            } rmi;
            struct {
                uint32_t scratch[2 * LSORT_MAX_TREE_DEV + 2];
                uint32_t wsum[NT / 32 + 1];
                uint64_t spl[LSORT_MAX_TREE_DEV];
            } tree;
        } u;
        uint64_t red64[NT / 32];
    };
};
using ModelSmall = ModelCfg<256, 2048>;
using ModelMid = ModelCfg<512, 8192>;

// Cell-table model (kModelLut, GPU policy) over the sorted sample A[0, s): cells of
// 2^shift keys from A[0], and cell c's bucket = floor(r_c * nb / s) with r_c the
// number of samples below the cell's start -- the sample's empirical CDF read at
// the cell starts (monotone; buckets are unions of cells). Cells
// (cell(A[i-1]), cell(A[i])] all have r = i, so thread i fills them: O(cells + s).
// Returns the largest bucket count of the sample itself (the quality check).
// hist: >= nb words of scratch.
template <int NT>
__device__ uint64_t build_lut_block(const uint64_t* A, uint32_t s, uint32_t nb, ModelHdr* h, uint8_t* payload,
                                    uint32_t* hist, uint64_t* red) {
    const uint32_t ncell = lut_model_cells(nb);
    const uint64_t smin = A[0];
    const uint32_t shift = lut_pick_shift(smin, A[s - 1], ncell);
    uint16_t* lut = (uint16_t*)payload;
    for (uint32_t i = threadIdx.x; i <= s; i += NT) {
        const uint32_t lo = i == 0 ? 0u : lut_cell(A[i - 1], smin, shift, ncell) + 1;
        const uint32_t hi = i == s ? ncell - 1 : lut_cell(A[i], smin, shift, ncell);
        const uint64_t v = (uint64_t)i * nb / s;
        const uint16_t b = (uint16_t)(v >= nb ? nb - 1 : v);
        for (uint32_t c = lo; c <= hi; ++c) lut[c] = b;
    }
    for (uint32_t b = threadIdx.x; b < nb; b += NT) hist[b] = 0;
    if (threadIdx.x == 0) {
        h->kind = kRadix;
        h->flags = kModelLut;
        h->nbuckets = nb;
        h->B = ncell;
        h->shift = shift;
        h->radix_min = smin;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < s; i += NT) atomicAdd(&hist[lut[lut_cell(A[i], smin, shift, ncell)]], 1u);
    __syncthreads();
    uint64_t mx = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += NT) mx = hist[b] > mx ? hist[b] : mx;
    return block_reduce_max<NT>(mx, red);
}

// Radix/fill fallback model: min/max of the whole segment (one CTA).
template <int NT>
__device__ void build_radix_model(const SegDesc& sd, const void* src, bool f64, ModelHdr* h, uint64_t* red) {
    uint64_t mn = ~0ull, mx = 0;
    for (uint64_t i = threadIdx.x; i < sd.n; i += NT) {
        uint64_t k = load_key(src, sd.in_begin + i, f64);
        mn = k < mn ? k : mn;
        mx = k > mx ? k : mx;
    }
    mn = block_reduce_min<NT>(mn, red);
    mx = block_reduce_max<NT>(mx, red);
    if (threadIdx.x == 0) {
        h->flags = 0;  // (not a cell table: the model record is reused memory)
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

// Draw sample draws [j0, j0+cnt) of the segment stream into shared A, sort.
template <bool IN_F64, class MC>
__device__ void sample_sorted(const SegDesc& sd, const void* src, uint64_t seed, uint32_t j0, uint32_t cnt,
                              typename MC::Smem& S, bool eq = false, const uint64_t* pre = nullptr) {
    constexpr int NT = sizeof(S.red64) / 8 * 32;
    if (pre) {  // drawn by a many-CTA gather (one SM cannot keep enough random loads in flight)
        for (uint32_t i = threadIdx.x; i < cnt; i += NT) S.sort.A[i] = pre[i];
    } else
    // random gather: 8 independent loads in flight per thread (a rolled loop
    // waits one DRAM latency per key)
    {
    const uint64_t minv = sd.n ? ~0ull / sd.n : 0ull;
    for (uint32_t i0 = threadIdx.x; i0 < cnt; i0 += 8 * NT) {
        uint64_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = i0 + u * NT;
            v[u] = i < cnt ? load_key(src, sd.in_begin + sample_index_inv(seed, j0 + i, sd.n, minv), IN_F64) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t i = i0 + u * NT;
            if (i < cnt) S.sort.A[i] = v[u];
        }
    }
    }
    __syncthreads();
    if (cnt > 1) {
        MC::SS::sort_fast(S.sort.A, cnt, S.sort, eq);  // -> S.sort.B
        for (uint32_t i = threadIdx.x; i < cnt; i += NT) S.sort.A[i] = S.sort.B[i];
    }
    __syncthreads();
}

// Alg. 5 build_partition_model for one segment. With
// aux != nullptr (first-sample-only mode for a big segment) the learned
// branch stops after the policy decision and builds the splitter tree that
// partitions the big RMI sample; *gate tells the following kernels which
// branch was taken.
template <bool IN_F64, class MC>
__device__ void build_model_cta(const SegDesc& sd, const void* src, uint8_t* models, const DevCfg& cfg,
                                typename MC::Smem& S, bool first_only, uint8_t* aux, uint32_t aux_budget,
                                uint32_t* gate, const uint64_t* pre = nullptr, uint32_t* dslices = nullptr) {
    constexpr int NT = sizeof(S.red64) / 8 * 32;
    ModelHdr* h = (ModelHdr*)(models + sd.model_off);
    uint8_t* payload = models + sd.model_off + sizeof(ModelHdr);
    if (sd.flags & kSegForceRadix) {
        build_radix_model<NT>(sd, src, IN_F64, h, S.red64);
        if (gate && threadIdx.x == 0) *gate = 0;
        return;
    }
    const uint64_t n = sd.n;
    const uint64_t seed = seg_seed(cfg.seed, sd.begin, sd.depth);
    // GPU policy: a child of the level-0 partition trains on its slice of the
    // parent's sorted sample (a uniform random sample of exactly its keys, of
    // the size the reference would draw) -- evenly thinned to the CTA's
    // capacity, still sorted: no gather, no sort
    const bool slice = cfg.psample != nullptr && sd.pslice != 0 && !first_only;
    uint32_t s1;
    if (slice) {
        const uint64_t off = sd.pslice >> 24;
        const uint32_t len = (uint32_t)(sd.pslice & 0xffffffu);
        s1 = min(len, (uint32_t)MC::kCap);
        for (uint32_t i = threadIdx.x; i < s1; i += NT)
            S.sort.A[i] = cfg.psample[off + (uint64_t)i * len / s1];
        __syncthreads();
    } else {
        s1 = (uint32_t)first_sample_size(cfg, n);
        // a root-level sample spans the whole key range: equalised digits
        sample_sorted<IN_F64, MC>(sd, src, seed, 0, s1, S, first_only || sd.depth == 0, first_only ? pre : nullptr);
    }
    const uint64_t* A = S.sort.A;
    uint64_t d = 0;
    for (uint32_t i = threadIdx.x + 1; i < s1; i += NT) d += A[i] != A[i - 1];
    d = block_reduce_sum_u64<NT>(d, S.red64);
    const uint64_t distinct = 1 + d;
    const double dup = __dsub_rn(1.0, __ddiv_rn((double)distinct, (double)s1));  // models.cpp:187-193
    const bool learned = n >= cfg.min_rmi_input && dup <= cfg.max_dup;
    if (threadIdx.x == 0) {
        h->dup = dup;
        h->s1 = s1;
        h->flags = 0;
        h->cdf_lo = 0.0;
        h->inv_span = 1.0;  // Learned::inv_span() with cdf [0,1] (models.hpp:134-137)
        if (gate) *gate = learned ? 1u : 0u;
    }
    if (learned) {
        const uint32_t s2 = slice ? s1 : (uint32_t)rmi_sample_size(cfg, n);
        if (threadIdx.x == 0) {
            h->kind = kLearned;
            h->nbuckets = sd.rmi_b;
            h->B = sd.rmi_b;
            h->s2 = s2;
        }
        if (first_only) {
            // splitter tree over the first sample: partitions the RMI sample
            tree_build_block<NT>(A, s1, aux_budget, true, (ModelHdr*)aux, aux + sizeof(ModelHdr),
                                 S.u.tree.scratch, S.u.tree.wsum, S.u.tree.spl);
            return;
        }
        __syncthreads();
        if (!slice) sample_sorted<IN_F64, MC>(sd, src, seed, s1, s2, S);
        if (cfg.lut && sd.depth >= 1) {  // GPU policy: cell table instead of an RMI
            const uint64_t mx = build_lut_block<NT>(A, s2, sd.rmi_b, h, payload, S.u.rmi.first, S.red64);
            if (poor_model(mx, s2, sd.rmi_b)) {
                if (threadIdx.x == 0) h->flags = 0;
                tree_build_block<NT>(A, s2, sd.tree_k, true, h, payload, S.u.tree.scratch, S.u.tree.wsum,
                                     S.u.tree.spl);
            }
            return;
        }
        train_rmi_block<NT>(A, s2, sd.rmi_b, h, (RmiEntry*)payload, S.u.rmi.first, S.u.rmi.lo, S.u.rmi.hi,
                            S.u.rmi.big, S.u.rmi.red);
        if (cfg.quality) {
            __syncthreads();
            uint32_t* hist = S.u.rmi.first;  // free after training
            Classifier Cl;
            Cl.init((const uint8_t*)h);
            for (uint32_t b = threadIdx.x; b < Cl.nb; b += NT) hist[b] = 0;
            __syncthreads();
            for (uint32_t i = threadIdx.x; i < s2; i += NT) atomicAdd(&hist[Cl.classify<kLearned>(A[i])], 1u);
            __syncthreads();
            uint64_t mx = 0;
            for (uint32_t b = threadIdx.x; b < Cl.nb; b += NT) mx = hist[b] > mx ? hist[b] : mx;
            mx = block_reduce_max<NT>(mx, S.red64);
            if (poor_model(mx, s2, Cl.nb))
                tree_build_block<NT>(A, s2, sd.tree_k, true, h, payload, S.u.tree.scratch, S.u.tree.wsum,
                                     S.u.tree.spl);
        }
    } else {
        if (threadIdx.x == 0) h->s2 = 0;
        tree_build_block<NT>(A, s1, sd.tree_k, true, h, payload, S.u.tree.scratch, S.u.tree.wsum, S.u.tree.spl);
        if (dslices) {  // a tree root: its buckets' offsets in the sorted first sample (one-pass level 0)
            __syncthreads();
            const MView m = model_view((const uint8_t*)h);
            const ModelHdr& th = *m.h;
            auto bk = [&](uint64_t x) {
                return tree_bucket(th.levels, th.leaf_origin, th.nsplit, m.tree, m.spl, m.eqo, x) & 0x7fffffffu;
            };
            for (uint32_t i = threadIdx.x; i <= s1; i += NT) {
                const uint32_t b = i < s1 ? bk(A[i]) : th.nbuckets;
                const uint32_t lo = i ? bk(A[i - 1]) + 1 : 0u;
                for (uint32_t q = lo; q <= b; ++q) dslices[q] = i;
            }
        }
    }
}

template <bool IN_F64, class MC, int NT>
__global__ void __launch_bounds__(NT, NT == 256 ? 3 : 1) k_build_models(const SegDesc* segs, const uint32_t* idx, const void* src,
                                                    uint8_t* models, DevCfg cfg) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    typename MC::Smem& S = *(typename MC::Smem*)smem_u4;
    const SegDesc sd = segs[idx[blockIdx.x]];
    build_model_cta<IN_F64, MC>(sd, src, models, cfg, S, false, nullptr, 0, nullptr);
}

template <bool IN_F64>
__global__ void __launch_bounds__(512, 1) k_first_sample(const uint64_t* pre, const SegDesc* seg, const void* src, uint8_t* models,
                                                     DevCfg cfg, uint8_t* aux, uint32_t aux_budget, uint32_t* gate,
                                                     uint32_t* dslices) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    ModelMid::Smem& S = *(ModelMid::Smem*)smem_u4;
    const SegDesc sd = *seg;
    build_model_cta<IN_F64, ModelMid>(sd, src, models, cfg, S, true, aux, aux_budget, gate, pre, dslices);
}

template <bool IN_F64>
__global__ void k_gather(const SegDesc* seg, const void* src, uint64_t seed, uint64_t j0, uint64_t s,
                         uint64_t* out, const uint32_t* gate) {
    griddep_wait();
    if (gate && *gate == 0) return;
    const SegDesc sd = *seg;
    const uint64_t minv = sd.n ? ~0ull / sd.n : 0ull;
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < s; j += (uint64_t)gridDim.x * blockDim.x)
        out[j] = load_key(src, sd.in_begin + sample_index_inv(seed, j0 + j, sd.n, minv), IN_F64);
}


// ============================================= multi-CTA RMI training
// Over a sorted sample in global memory. Every kernel takes `gate` (nullptr
// = always run): 0 means the segment's policy chose the splitter tree and the
// kernel exits at once (big-segment pipeline, no host round trip).
// Workspace layout: [part: 4 * nch doubles][root: 8 doubles][first: B+1 u32]
constexpr int kTrainChunk = 4096;
constexpr int kTrainNT = 256;

struct TrainWS {
    double* part;   // [4][nch]: sx, sy, sxx, sxy per chunk
    double* root;   // rs, ri, base, scale, mx, my
    double* big;    // [B][kBigSplit][3] partial sums of the big-slice fits
    uint32_t* first;
    uint32_t* bigcnt;  // [B] arrival counters (wrap to 0)
    uint32_t nch;
};
constexpr int kBigSplitWS = 16;
__host__ __device__ inline TrainWS train_ws(void* ws, uint64_t s, uint32_t B) {
    TrainWS w;
    w.nch = (uint32_t)((s + kTrainChunk - 1) / kTrainChunk);
    w.part = (double*)ws;
    w.root = w.part + 4 * (size_t)w.nch;
    w.big = w.root + 8;
    w.first = (uint32_t*)(w.big + (size_t)B * kBigSplitWS * 3);
    w.bigcnt = w.first + B + 2;
    return w;
}
size_t train_workspace_bytes(uint64_t s, uint32_t B) {
    uint64_t nch = (s + kTrainChunk - 1) / kTrainChunk;
    return 8 * (4 * nch + 8) + 24 * (size_t)B * kBigSplitWS + 4 * ((size_t)B + 2) + 4 * (size_t)B;
}
__device__ __forceinline__ bool gated_off(const uint32_t* gate) { return gate && *gate == 0; }

__device__ __forceinline__ void base_scale(const uint64_t* s, uint32_t n, double& base, double& scale) {
    base = __ull2double_rn(s[0]);
    const double kmax = __ull2double_rn(s[n - 1]);
    scale = kmax > base ? __ddiv_rn(1.0, __dsub_rn(kmax, base)) : 0.0;  // models.cpp:47-49
}

// pass 1 (PASS2 = false): per-chunk sum of xn and target i/n;
// pass 2 (PASS2 = true): per-chunk centred sums (models.cpp:26-31)
template <bool PASS2>
__global__ void __launch_bounds__(kTrainNT) k_train_sums(const uint64_t* s, uint32_t n, void* wsp, uint32_t B,
                                                        const uint32_t* gate) {
    griddep_wait();
    __shared__ double red[kTrainNT / 32];
    if (gated_off(gate)) return;
    TrainWS w = train_ws(wsp, n, B);
    double base, scale;
    base_scale(s, n, base, scale);
    const double nd = (double)n;
    const uint32_t c0 = blockIdx.x * kTrainChunk;
    const uint32_t per = kTrainChunk / kTrainNT;
    const uint32_t lo = min(n, c0 + threadIdx.x * per), hi = min(n, lo + per);
    double a = 0.0, b = 0.0;
    if (!PASS2) {
        for (uint32_t i = lo; i < hi; ++i) {
            a = __dadd_rn(a, rmi_normalize(base, scale, s[i]));
            b = __dadd_rn(b, __ddiv_rn((double)i, nd));
        }
    } else {
        const double mx = w.root[4], my = w.root[5];
        for (uint32_t i = lo; i < hi; ++i) {
            double dx = __dsub_rn(rmi_normalize(base, scale, s[i]), mx);
            a = __dadd_rn(a, __dmul_rn(dx, dx));
            b = __dadd_rn(b, __dmul_rn(dx, __dsub_rn(__ddiv_rn((double)i, nd), my)));
        }
    }
    a = block_sum_f64<kTrainNT>(a, red);
    b = block_sum_f64<kTrainNT>(b, red);
    if (threadIdx.x == 0) {
        w.part[(PASS2 ? 2 : 0) * (size_t)w.nch + blockIdx.x] = a;
        w.part[(PASS2 ? 3 : 1) * (size_t)w.nch + blockIdx.x] = b;
    }
}

// fixed-order reduction of the chunk partials (one CTA)
template <bool PASS2>
__global__ void __launch_bounds__(kTrainNT) k_train_reduce(const uint64_t* s, uint32_t n, void* wsp, uint32_t B,
                                                          const uint32_t* gate) {
    griddep_wait();
    __shared__ double red[kTrainNT / 32];
    if (gated_off(gate)) return;
    TrainWS w = train_ws(wsp, n, B);
    const uint32_t per = (w.nch + kTrainNT - 1) / kTrainNT;
    const uint32_t lo = min(w.nch, threadIdx.x * per), hi = min(w.nch, lo + per);
    const double* pa = w.part + (PASS2 ? 2 : 0) * (size_t)w.nch;
    const double* pb = w.part + (PASS2 ? 3 : 1) * (size_t)w.nch;
    double a = 0.0, b = 0.0;
    for (uint32_t i = lo; i < hi; ++i) {
        a = __dadd_rn(a, pa[i]);
        b = __dadd_rn(b, pb[i]);
    }
    a = block_sum_f64<kTrainNT>(a, red);
    b = block_sum_f64<kTrainNT>(b, red);
    if (threadIdx.x == 0) {
        const double nd = (double)n;
        if (!PASS2) {
            w.root[4] = __ddiv_rn(a, nd);  // mx
            w.root[5] = __ddiv_rn(b, nd);  // my
        } else {
            const double mx = w.root[4], my = w.root[5];
            double rs, ri;
            if (!(a > 0.0)) { rs = 0.0; ri = my; }
            else {
                double sl = __ddiv_rn(b, a);
                if (sl < 0.0) { rs = 0.0; ri = my; }
                else { rs = sl; ri = __dsub_rn(my, __dmul_rn(sl, mx)); }
            }
            double base, scale;
            base_scale(s, n, base, scale);
            w.root[0] = rs;
            w.root[1] = ri;
            w.root[2] = base;
            w.root[3] = scale;
        }
    }
}

// Slice boundaries in one coalesced pass: element i (route r_i, nondecreasing
// along the sorted sample) writes first[m] = i for every m in (r_{i-1}, r_i];
// the last element also closes (r_last, B]. Each first[m] is written once.
__global__ void __launch_bounds__(kTrainNT) k_train_bounds(const uint64_t* s, uint32_t n, void* wsp, uint32_t B,
                                                          const uint32_t* gate) {
    griddep_wait();
    if (gated_off(gate)) return;
    TrainWS w = train_ws(wsp, n, B);
    const double rs = w.root[0], ri = w.root[1], base = w.root[2], scale = w.root[3];
    for (uint32_t i = blockIdx.x * kTrainNT + threadIdx.x; i < n; i += gridDim.x * kTrainNT) {
        const uint32_t r = rmi_route(rs, ri, B, rmi_normalize(base, scale, s[i]));
        const uint32_t rp = i == 0 ? 0u : rmi_route(rs, ri, B, rmi_normalize(base, scale, s[i - 1])) + 1;
        for (uint32_t m = (i == 0 ? 0u : rp); m <= r; ++m) w.first[m] = i;
        if (i == n - 1)
            for (uint32_t m = r + 1; m <= B; ++m) w.first[m] = n;
    }
}

// Sequential fit_line of every slice <= kSeqFitMax samples (bit-exact, the
// reference's summation order): one warp per submodel stages xn and the
// targets in shared memory (parallel, coalesced), then one lane runs the
// dependent add chains.
constexpr int kFitWarps = 4;
constexpr int kMedFitMax = 16384;  // slices up to this: one warp (k_train_fits); above: k_train_bigfits
__global__ void __launch_bounds__(32 * kFitWarps) k_train_fits(const uint64_t* s, uint32_t n, void* wsp, uint32_t B,
                                                              RmiEntry* E, const uint32_t* gate) {
    griddep_wait();
    __shared__ double xs[kFitWarps][kSeqFitMax];
    __shared__ double ys[kFitWarps][kSeqFitMax];
    if (gated_off(gate)) return;
    TrainWS w = train_ws(wsp, n, B);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t m = blockIdx.x * kFitWarps + warp;
    if (m >= B) return;
    const uint32_t f = min(w.first[m], n), l = min(max(w.first[m + 1], f), n);
    const uint32_t len = l - f;
    if (len == 0 || len > (uint32_t)kMedFitMax) return;
    const double base = w.root[2], scale = w.root[3], nd = (double)n;
    if (len > (uint32_t)kSeqFitMax) {
        // medium slice: shifted one-pass sums, lane-strided, fixed shuffle
        // tree -> deterministic, within the test tolerance (as k_train_bigfits)
        const double c = rmi_normalize(base, scale, s[f]);
        double sd = 0.0, sdd = 0.0, sde = 0.0;
        for (uint32_t i = f + lane; i < l; i += 32) {
            const double dd = __dsub_rn(rmi_normalize(base, scale, s[i]), c);
            const double e = (double)(i - f);
            sd = __dadd_rn(sd, dd);
            sdd = __dadd_rn(sdd, __dmul_rn(dd, dd));
            sde = __dadd_rn(sde, __dmul_rn(dd, e));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sd = __dadd_rn(sd, __shfl_xor_sync(FULL_MASK, sd, o));
            sdd = __dadd_rn(sdd, __shfl_xor_sync(FULL_MASK, sdd, o));
            sde = __dadd_rn(sde, __shfl_xor_sync(FULL_MASK, sde, o));
        }
        if (lane == 0) {
            const double cn = (double)len;
            const double md = __ddiv_rn(sd, cn);
            const double mx = __dadd_rn(c, md);
            const double me = __dmul_rn(0.5, (double)(len - 1));
            const double my = __ddiv_rn(__dadd_rn((double)f, me), nd);
            const double sxx = __dsub_rn(sdd, __dmul_rn(sd, md));
            const double sxy = __ddiv_rn(__dsub_rn(sde, __dmul_rn(sd, me)), nd);
            double sl = 0.0, ic = my;  // models.cpp:32-34
            if (sxx > 0.0) {
                const double q = __ddiv_rn(sxy, sxx);
                if (!(q < 0.0)) { sl = q; ic = __dsub_rn(my, __dmul_rn(q, mx)); }
            }
            E[m].slope = sl;
            E[m].intercept = ic;
        }
        return;
    }
    double* x = xs[warp];
    double* y = ys[warp];
    for (uint32_t j = lane; j < len; j += 32) {
        x[j] = rmi_normalize(base, scale, s[f + j]);
        y[j] = __ddiv_rn((double)(f + j), nd);
    }
    __syncwarp();
    double sx = 0.0, sy = 0.0;
    if (lane == 0)
        for (uint32_t j = 0; j < len; ++j) { sx = __dadd_rn(sx, x[j]); sy = __dadd_rn(sy, y[j]); }
    const double mx = __shfl_sync(FULL_MASK, __ddiv_rn(sx, (double)len), 0);
    const double my = __shfl_sync(FULL_MASK, __ddiv_rn(sy, (double)len), 0);
    for (uint32_t j = lane; j < len; j += 32) {  // products in parallel, sums in order below
        const double dx = __dsub_rn(x[j], mx);
        x[j] = __dmul_rn(dx, dx);
        y[j] = __dmul_rn(dx, __dsub_rn(y[j], my));
    }
    __syncwarp();
    if (lane == 0) {
        double sxx = 0.0, sxy = 0.0;
        for (uint32_t j = 0; j < len; ++j) { sxx = __dadd_rn(sxx, x[j]); sxy = __dadd_rn(sxy, y[j]); }
        double sl = 0.0, ic = my;  // models.cpp:32-34
        if (sxx > 0.0) {
            double q = __ddiv_rn(sxy, sxx);
            if (!(q < 0.0)) { sl = q; ic = __dsub_rn(my, __dmul_rn(q, mx)); }
        }
        E[m].slope = sl;
        E[m].intercept = ic;
    }
}

// Slices larger than kSeqFitMax: kBigSplit CTAs per slice, one pass of
// shifted sums (d = xn - xn(first), e = i - first) so no division sits in the
// loop; the last CTA of a slice (atomicInc counter, wraps back to 0) combines
// the partials in a fixed order -> deterministic. Within RMI_RTOL of the
// reference's sequential sums (models.cpp:14-35).
constexpr int kBigFitNT = 256;
constexpr int kBigSplit = 16;
__global__ void __launch_bounds__(kBigFitNT) k_train_bigfits(const uint64_t* s, uint32_t n, void* wsp, uint32_t B,
                                                            RmiEntry* E, const uint32_t* gate) {
    griddep_wait();
    __shared__ double red[kBigFitNT / 32];
    __shared__ uint32_t last;
    if (gated_off(gate)) return;
    TrainWS w = train_ws(wsp, n, B);
    for (uint32_t item = blockIdx.x; item < B * kBigSplit; item += gridDim.x) {
    const uint32_t m = item / kBigSplit, ysp = item % kBigSplit;
    const uint32_t f = min(w.first[m], n), l = min(max(w.first[m + 1], f), n);
    if (l - f <= (uint32_t)kMedFitMax) continue;
    const double base = w.root[2], scale = w.root[3];
    const uint32_t cnt = l - f;
    const double c = rmi_normalize(base, scale, s[f]);
    double sd = 0.0, sdd = 0.0, sde = 0.0;
    for (uint32_t i = f + ysp * kBigFitNT + threadIdx.x; i < l; i += kBigSplit * kBigFitNT) {
        const double d = __dsub_rn(rmi_normalize(base, scale, s[i]), c);
        const double e = (double)(i - f);
        sd = __dadd_rn(sd, d);
        sdd = __dadd_rn(sdd, __dmul_rn(d, d));
        sde = __dadd_rn(sde, __dmul_rn(d, e));
    }
    sd = block_sum_f64<kBigFitNT>(sd, red);
    sdd = block_sum_f64<kBigFitNT>(sdd, red);
    sde = block_sum_f64<kBigFitNT>(sde, red);
    double* part = w.big + ((size_t)m * kBigSplit + ysp) * 3;
    if (threadIdx.x == 0) {
        part[0] = sd;
        part[1] = sdd;
        part[2] = sde;
        __threadfence();
        last = atomicInc(&w.bigcnt[m], kBigSplit - 1) == kBigSplit - 1;
    }
    __syncthreads();
    const bool fin = last;
    __syncthreads();  // `last` is rewritten by the next item
    if (!fin || threadIdx.x != 0) continue;
    __threadfence();
    const volatile double* P = w.big + (size_t)m * kBigSplit * 3;
    double Sd = 0.0, Sdd = 0.0, Sde = 0.0;
    for (int q = 0; q < kBigSplit; ++q) {
        Sd = __dadd_rn(Sd, P[3 * q]);
        Sdd = __dadd_rn(Sdd, P[3 * q + 1]);
        Sde = __dadd_rn(Sde, P[3 * q + 2]);
    }
    const double cn = (double)cnt, nd = (double)n;
    const double md = __ddiv_rn(Sd, cn);
    const double mx = __dadd_rn(c, md);
    const double me = __dmul_rn(0.5, (double)(cnt - 1));            // mean of e, exact
    const double my = __ddiv_rn(__dadd_rn((double)f, me), nd);      // mean of i/n
    const double sxx = __dsub_rn(Sdd, __dmul_rn(Sd, md));           // sum (x - mx)^2
    const double sxy = __ddiv_rn(__dsub_rn(Sde, __dmul_rn(Sd, me)), nd);  // sum (x - mx)(y - my)
    double sl = 0.0, ic = my;  // models.cpp:32-34
    if (sxx > 0.0) {
        double q = __ddiv_rn(sxy, sxx);
        if (!(q < 0.0)) { sl = q; ic = __dsub_rn(my, __dmul_rn(q, mx)); }
    }
    E[m].slope = sl;
    E[m].intercept = ic;
    }
}

// enforce_monotonic (models.cpp:101-126) + header + compiled table, one CTA
constexpr int kEnforceNT = 1024;
__global__ void __launch_bounds__(kEnforceNT) k_train_enforce(const uint64_t* s, uint32_t n, void* wsp, uint32_t B,
                                                             uint8_t* model, uint32_t nbuckets, const uint32_t* gate) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    double* lo = (double*)smem_u4;
    double* hi = lo + B;
    __shared__ double red[2 * (kEnforceNT / 32)];
    if (gated_off(gate)) return;
    TrainWS w = train_ws(wsp, n, B);
    ModelHdr* h = (ModelHdr*)model;
    RmiEntry* E = (RmiEntry*)(model + sizeof(ModelHdr));
    const double base = w.root[2], scale = w.root[3];
    for (uint32_t m = threadIdx.x; m < B; m += kEnforceNT) {
        uint32_t f = min(w.first[m], n), l = min(w.first[m + 1], n);
        if (l > f) {
            double sl = E[m].slope, ic = E[m].intercept;
            lo[m] = __dadd_rn(__dmul_rn(sl, rmi_normalize(base, scale, s[f])), ic);
            hi[m] = __dadd_rn(__dmul_rn(sl, rmi_normalize(base, scale, s[l - 1])), ic);
        } else {
            lo[m] = -INFINITY;
            hi[m] = INFINITY;
        }
    }
    __syncthreads();
    block_fold_scan<kEnforceNT>(lo, B, false, red, StepMax());
    block_fold_scan<kEnforceNT>(hi, B, true, red, StepMin());
    for (uint32_t m = threadIdx.x; m < B; m += kEnforceNT) {
        double hh = hi[m];
        if (m + 1 < B) hh = dmin_ref(hh, lo[m + 1]);
        hh = dmax_ref(hh, lo[m]);
        double ll = dclamp01(lo[m]);
        hh = dclamp01(hh);
        if (m == 0) ll = 0.0;
        if (m == B - 1) hh = 1.0;
        if (min(w.first[m + 1], n) <= min(w.first[m], n)) {
            E[m].slope = 0.0;
            E[m].intercept = __dmul_rn(0.5, __dadd_rn(ll, hh));
        }
        E[m].lo = ll;
        E[m].hi = hh;
    }
    if (threadIdx.x == 0) {
        h->kind = kLearned;
        h->nbuckets = nbuckets;
        h->B = B;
        h->root_slope = w.root[0];
        h->root_icpt = w.root[1];
        h->key_base = base;
        h->key_scale = scale;
        h->cdf_lo = 0.0;
        h->inv_span = 1.0;
    }
    __syncthreads();
    compile_learned(model, threadIdx.x, kEnforceNT);
}

__global__ void __launch_bounds__(512) k_tree_build(const uint64_t* sorted, uint32_t s, uint32_t budget,
                                                   int eq_mode, uint8_t* model) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    ModelMid::Smem& S = *(ModelMid::Smem*)smem_u4;
    for (uint32_t i = threadIdx.x; i < s; i += 512) S.sort.A[i] = sorted[i];
    __syncthreads();
    tree_build_block<512>(S.sort.A, s, budget, eq_mode != 0, (ModelHdr*)model, model + sizeof(ModelHdr),
                          S.u.tree.scratch, S.u.tree.wsum, S.u.tree.spl);
}

__global__ void __launch_bounds__(512) k_block_sort(uint64_t* keys, uint32_t n) {
    griddep_wait();
    extern __shared__ uint4 smem_u4[];
    ModelMid::Smem& S = *(ModelMid::Smem*)smem_u4;
    for (uint32_t i = threadIdx.x; i < n; i += 512) S.sort.A[i] = keys[i];
    __syncthreads();
    if (n > 1) {
        ModelMid::SS::sort_fast(S.sort.A, n, S.sort);
        for (uint32_t i = threadIdx.x; i < n; i += 512) S.sort.A[i] = S.sort.B[i];
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += 512) keys[i] = S.sort.A[i];
}

// ------------------------------------------------ model quality (GPU policy)
// One CTA: if the model is poor (poor_model: largest bucket share), replace
// the learned model by a splitter tree over the same sorted sample.
// (bucket sizes = differences of the sample's bucket offsets; *redo = 1 when
// the model was replaced, so the offsets are recomputed for the tree)
__global__ void __launch_bounds__(512) k_quality(const uint64_t* s, uint32_t n, uint8_t* model, uint32_t tree_k,
                                                 const uint32_t* offs, uint32_t* redo, const uint32_t* gate,
                                                 uint32_t share_den, uint32_t poor_share) {
    griddep_wait();
    __shared__ uint32_t scratch[2 * LSORT_MAX_TREE_DEV + 2];
    __shared__ uint32_t wsum[512 / 32 + 1];
    __shared__ uint64_t spl[LSORT_MAX_TREE_DEV];
    __shared__ uint64_t red[512 / 32];
    if (threadIdx.x == 0) *redo = 0;
    if (gated_off(gate)) return;
    ModelHdr* h = (ModelHdr*)model;
    if (h->kind != kLearned) return;
    const uint32_t nb = h->nbuckets;
    uint64_t mx = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += 512) {
        const uint32_t c = offs[b + 1] - offs[b];
        mx = c > mx ? c : mx;
    }
    mx = block_reduce_max<512>(mx, red);
    const bool poor = mx * poor_share > n && mx * nb > (uint64_t)kPoorMean * n;
    if (!poor && !(share_den && mx * share_den > n)) return;
    tree_build_block<512>(s, n, tree_k, true, h, model + sizeof(ModelHdr), scratch, wsum, spl);
    if (threadIdx.x == 0) *redo = 1;
}

size_t quality_workspace_bytes() { return 4 * ((size_t)LSORT_MAX_RMI_DEV + 8); }

// ---------------------------------------------- root cell table (GPU policy)
// A learned root's RMI is replaced by a cell-table model (kModelLut) over its
// sorted sample when the table balances the sample at least as evenly as the
// bound below: one u16 read per key in the one-pass level 0 instead of an RMI
// evaluation (root route + 20-byte submodel lookup, ~30 instructions).
// (1) k_lut_ranks (many CTAs): R[c] = number of samples below the start of cell c;
// (2) k_root_lut (one CTA): lut[c] = min(nb - 1, R[c] nb / s), the sample's
//     bucket sizes from R at the first cell of every bucket; accepted if the
//     largest holds <= 2x the mean -- then header + table replace the RMI.
__device__ __forceinline__ void lut_geometry(const uint64_t* s, uint32_t n, uint32_t ncell, uint64_t& origin,
                                             uint32_t& shift) {
    origin = s[0];
    shift = lut_pick_shift(origin, s[n - 1], ncell);
}
// skip_sign: float keys whose sample spans both signs -- a linear table over that
// encoded range (>= 2^63 keys) cannot balance them; only the log table is tried
__global__ void __launch_bounds__(256) k_lut_ranks(const uint64_t* s, uint32_t n, const uint8_t* model, uint32_t* R,
                                                   const uint32_t* gate, uint32_t skip_sign) {
    griddep_wait();
    if (gated_off(gate)) return;
    const ModelHdr* h = (const ModelHdr*)model;
    if (h->kind != kLearned || n < 2) return;
    if (skip_sign && ((s[0] ^ s[n - 1]) >> 63)) return;
    const uint32_t ncell = min(kRootLutCells, kLutModelCellsPerBucket * h->B);
    uint64_t origin;
    uint32_t shift;
    lut_geometry(s, n, ncell, origin, shift);
    // one lower-bound search per cell (a per-sample fill of the cells between
    // consecutive samples leaves one thread thousands of cells across a gap)
    for (uint32_t c = blockIdx.x * 256 + threadIdx.x; c < ncell; c += gridDim.x * 256) {
        const uint64_t start = lut_cell_start(c, origin, shift);
        uint32_t b = 0, m = n;
        while (m > 0) {
            const uint32_t h = m >> 1;
            if (s[b + h] < start) { b += h + 1; m -= h + 1; }
            else m = h;
        }
        R[c] = c ? b : 0u;
    }
}
// Log tables (when the linear table is rejected): (3) k_binade_starts (many
// CTAs): first sample index of every binade of the sample's span; (4)
// k_log_tab (one CTA): 2^floor(log2(cells/2 x share)) cells per non-empty
// binade, entries by exclusive scan; (5) k_lut_fill (many CTAs): R per cell,
// cells (cell(s[i-1]), cell(s[i])] get i -- the cells follow the sample's
// density, so no thread walks a long gap; (6) k_root_lut in log mode.
struct LogWS {
    uint32_t* R;       // [kRootLutCells]
    uint32_t* bst;     // [kLogTabMax + 1]
    uint16_t* tab;     // [kLogTabMax]
    uint32_t* ncell;   // 0: rejected
};
__host__ __device__ inline LogWS log_ws(void* w) {
    LogWS L;
    L.R = (uint32_t*)w;
    L.bst = L.R + kRootLutCells;
    L.tab = (uint16_t*)(L.bst + kLogTabMax + 1);
    L.ncell = (uint32_t*)(L.tab + kLogTabMax);
    return L;
}
__global__ void __launch_bounds__(256) k_binade_starts(const uint64_t* s, uint32_t n, LogWS w, const uint32_t* gate) {
    griddep_wait();
    if (gated_off(gate) || n < 2) return;
    const uint32_t bmin = (uint32_t)(s[0] >> 52), ntab = (uint32_t)(s[n - 1] >> 52) - bmin + 1;
    if (ntab > kLogTabMax) return;
    for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i <= n; i += gridDim.x * 256) {
        const uint32_t b = i < n ? (uint32_t)(s[i] >> 52) - bmin : ntab;
        const uint32_t lo = i ? (uint32_t)(s[i - 1] >> 52) - bmin + 1 : 0u;
        for (uint32_t j = lo; j <= b; ++j) w.bst[j] = i;
    }
}
constexpr int kRootLutNT = 1024;
__global__ void __launch_bounds__(kRootLutNT) k_log_tab(const uint64_t* s, uint32_t n, LogWS w, const uint32_t* gate) {
    griddep_wait();
    __shared__ uint32_t cells[kLogTabMax];
    __shared__ uint32_t wsum[kRootLutNT / 32 + 1];
    if (gated_off(gate) || n < 2) return;
    const uint32_t bmin = (uint32_t)(s[0] >> 52), ntab = (uint32_t)(s[n - 1] >> 52) - bmin + 1;
    if (ntab > kLogTabMax) {
        if (threadIdx.x == 0) *w.ncell = 0;
        return;
    }
    uint32_t kk[kLogTabMax / kRootLutNT];
#pragma unroll
    for (uint32_t q = 0; q < kLogTabMax / kRootLutNT; ++q) {
        const uint32_t j = threadIdx.x + q * kRootLutNT;
        uint32_t c = 0, k = 0;
        if (j < ntab) {
            const uint32_t cnt = w.bst[j + 1] - w.bst[j];
            if (cnt) {
                const uint64_t want = (uint64_t)(kBinadeCells - 256) * cnt / n;
                k = want > 1 ? min(12u, 63u - (uint32_t)__clzll((long long)want)) : 0u;
                c = 1u << k;
            }
        }
        cells[j] = c;
        kk[q] = k;
    }
    __syncthreads();
    const uint32_t total = block_exclusive_scan_u32<kRootLutNT>(cells, kLogTabMax, wsum);
    if (threadIdx.x == 0) *w.ncell = total <= kBinadeCells ? total : 0u;
#pragma unroll
    for (uint32_t q = 0; q < kLogTabMax / kRootLutNT; ++q) {
        const uint32_t j = threadIdx.x + q * kRootLutNT;
        if (j < ntab) w.tab[j] = (uint16_t)((cells[j] & 0xfffu) | (kk[q] << 12));
    }
}
__global__ void __launch_bounds__(256) k_lut_fill(const uint64_t* s, uint32_t n, LogWS w, const uint32_t* gate) {
    griddep_wait();
    if (gated_off(gate) || n < 2 || *w.ncell == 0) return;
    const uint32_t ncell = *w.ncell;
    const uint32_t bmin = (uint32_t)(s[0] >> 52), ntab = (uint32_t)(s[n - 1] >> 52) - bmin + 1;
    for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i <= n; i += gridDim.x * 256) {
        const uint32_t c = i < n ? binade_cell(s[i], w.tab, bmin, ntab, ncell) : ncell - 1;
        const uint32_t lo = i ? binade_cell(s[i - 1], w.tab, bmin, ntab, ncell) + 1 : 0u;
        const uint32_t r = i < n ? i : n;
        for (uint32_t q = lo; q <= c; ++q) w.R[q] = r;
    }
}
__global__ void __launch_bounds__(kRootLutNT) k_root_lut(const uint64_t* s, uint32_t n, uint8_t* model,
                                                        const uint32_t* R, const uint32_t* gate, uint32_t* train_gate,
                                                        LogWS lw, uint32_t logm, uint32_t skip_sign) {
    griddep_wait();
    __shared__ uint32_t off[LSORT_MAX_RMI_DEV + 1];
    __shared__ uint64_t red[kRootLutNT / 32];
    // the RMI is trained (train_gate) unless the table is accepted
    const bool on = !gated_off(gate);
    if (threadIdx.x == 0) *train_gate = on ? 1u : 0u;
    if (!on) return;
    ModelHdr* h = (ModelHdr*)model;
    if (h->kind != kLearned || n < 2) return;
    if (logm && *lw.ncell == 0) return;  // no log table (too many binades or cells)
    if (!logm && skip_sign && ((s[0] ^ s[n - 1]) >> 63)) return;  // (k_lut_ranks)
    const uint32_t nb = h->nbuckets;
    const uint32_t ncell = logm ? *lw.ncell : min(kRootLutCells, kLutModelCellsPerBucket * h->B);
    uint64_t origin;
    uint32_t shift;
    lut_geometry(s, n, ncell, origin, shift);
    auto bucket = [&](uint32_t c) -> uint32_t {
        const uint64_t v = (uint64_t)R[c] * nb / n;
        return v >= nb ? nb - 1 : (uint32_t)v;
    };
    // off[b] = samples below bucket b's first cell (buckets no cell maps to: empty)
    for (uint32_t b = threadIdx.x; b <= nb; b += kRootLutNT) off[b] = n;
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < ncell; c += kRootLutNT) {
        const uint32_t b = bucket(c), lo = c == 0 ? 0u : bucket(c - 1) + 1;
        for (uint32_t q = lo; q <= b; ++q) off[q] = R[c];
    }
    __syncthreads();
    uint64_t mx = 0;
    for (uint32_t b = threadIdx.x; b < nb; b += kRootLutNT) {
        const uint32_t c = off[b + 1] - off[b];
        mx = c > mx ? c : mx;
    }
    mx = block_reduce_max<kRootLutNT>(mx, red);
    if (mx * nb > 2ull * n) return;  // keep the RMI
    uint16_t* lut = (uint16_t*)(model + sizeof(ModelHdr));
    uint32_t ntab = 0;
    if (logm) {  // log table: binade entries first
        const uint32_t bmin = (uint32_t)(s[0] >> 52);
        ntab = (uint32_t)(s[n - 1] >> 52) - bmin + 1;
        for (uint32_t j = threadIdx.x; j < ntab; j += kRootLutNT) lut[j] = lw.tab[j];
        lut += (ntab + 7) & ~7u;
        origin = bmin;
    }
    for (uint32_t c = threadIdx.x; c < ncell; c += kRootLutNT) lut[c] = (uint16_t)bucket(c);
    if (threadIdx.x == 0) {
        h->kind = kRadix;
        h->flags = logm ? (kModelLut | kModelLog) : kModelLut;
        h->B = ncell;
        h->levels = ntab;
        h->shift = shift;
        h->radix_min = origin;
        *train_gate = 0;
    }
}

size_t root_lut_workspace_bytes() {
    return 4 * (size_t)kRootLutCells + 4 * ((size_t)kLogTabMax + 1) + 2 * (size_t)kLogTabMax + 16;
}

void launch_root_lut(const uint64_t* sorted, uint64_t s, uint8_t* model, void* ws, const uint32_t* gate,
                     uint32_t* train_gate, cudaStream_t st, bool log_table, bool log_first) {
    const int g = (int)(kRootLutCells / 256);
    const LogWS w = log_ws(ws);
    const int gs = (int)std::min<uint64_t>((s + 2047) / 2048, (uint64_t)num_sms() * 2);
    auto log_try = [&](const uint32_t* gt) {  // gt: run only while *gt != 0
        pdl(k_binade_starts, gs, 256, 0, st, sorted, (uint32_t)s, w, gt);
        pdl(k_log_tab, 1, kRootLutNT, 0, st, sorted, (uint32_t)s, w, gt);
        pdl(k_lut_fill, gs, 256, 0, st, sorted, (uint32_t)s, w, gt);
        pdl(k_root_lut, 1, kRootLutNT, 0, st, sorted, (uint32_t)s, model, (const uint32_t*)w.R, gt, train_gate, w, 1u,
            0u);
    };
    auto lin_try = [&](const uint32_t* gt) {
        const uint32_t ss = log_table ? 1u : 0u;
        pdl(k_lut_ranks, g, 256, 0, st, sorted, (uint32_t)s, (const uint8_t*)model, (uint32_t*)ws, gt, ss);
        pdl(k_root_lut, 1, kRootLutNT, 0, st, sorted, (uint32_t)s, model, (const uint32_t*)ws, gt, train_gate, w, 0u, ss);
    };
    if (log_table && log_first) {
        log_try(gate);
        lin_try(train_gate);  // (the log table rejected: train_gate still 1)
        return;
    }
    lin_try(gate);
    if (log_table) log_try(train_gate);  // the linear table rejected (train_gate still 1)
}

// Bucket boundaries in a sorted sample (monotone bucket function): element i
// writes offsets[b] = i for every b in (bucket(s[i-1]), bucket(s[i])].
__global__ void __launch_bounds__(256) k_sample_slices(const uint64_t* s, uint32_t n, const uint8_t* model,
                                                       uint32_t* off, const uint32_t* gate) {
    griddep_wait();
    if (gated_off(gate)) return;
    Classifier Cl;
    Cl.init(model);
    const uint32_t nb = Cl.nb;
    for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += gridDim.x * 256) {
        const uint32_t bi = Cl.classify_any(s[i]) & 0x7fffffffu;
        const uint32_t lo = i == 0 ? 0u : (Cl.classify_any(s[i - 1]) & 0x7fffffffu) + 1;
        for (uint32_t b = lo; b <= bi; ++b) off[b] = i;
        if (i == n - 1)
            for (uint32_t b = bi + 1; b <= nb; ++b) off[b] = n;
    }
}

void launch_sample_slices(const uint64_t* sorted, uint64_t s, const uint8_t* model, uint32_t* offsets,
                          uint32_t nb_cap, const uint32_t* gate, cudaStream_t st) {
    (void)nb_cap;
    const int g = (int)std::min<uint64_t>((s + 1023) / 1024, (uint64_t)num_sms() * 4);
    pdl(k_sample_slices, g, 256, 0, st, sorted, (uint32_t)s, model, offsets, gate);
}



void launch_quality_check(const uint64_t* sorted, uint64_t s, uint8_t* model, uint32_t tree_k, void* ws,
                          uint32_t* offs, const uint32_t* gate, cudaStream_t st, uint32_t share_den,
                          uint32_t poor_share) {
    uint32_t* o = offs ? offs : (uint32_t*)ws;
    uint32_t* redo = (uint32_t*)ws + LSORT_MAX_RMI_DEV + 4;
    launch_sample_slices(sorted, s, model, o, 0, gate, st);
    pdl(k_quality, 1, 512, 0, st, sorted, (uint32_t)s, model, tree_k, o, redo, gate, share_den, poor_share);
    if (offs) launch_sample_slices(sorted, s, model, o, 0, redo, st);  // the tree's offsets
}

// ------------------------------------------------------------- launchers
void models_init(int optin) {
    allow_smem(k_build_models<true, ModelSmall, 256>, optin);
    allow_smem(k_build_models<false, ModelSmall, 256>, optin);
    allow_smem(k_build_models<true, ModelMid, 512>, optin);
    allow_smem(k_build_models<false, ModelMid, 512>, optin);
    allow_smem(k_first_sample<true>, optin);
    allow_smem(k_first_sample<false>, optin);
    allow_smem(k_train_enforce, optin);
    allow_smem(k_tree_build, optin);
    allow_smem(k_block_sort, optin);
}

void launch_build_models(const SegDesc* segs, const uint32_t* idx, uint32_t count, const void* src, int in_f64,
                         uint8_t* models, const DevCfg& cfg, int mid, cudaStream_t st) {
    if (!count) return;
    if (mid) {
        size_t sm = sizeof(ModelMid::Smem);
        if (in_f64) pdl(k_build_models<true, ModelMid, 512>, count, 512, sm, st, segs, idx, src, models, cfg);
        else pdl(k_build_models<false, ModelMid, 512>, count, 512, sm, st, segs, idx, src, models, cfg);
    } else {
        size_t sm = sizeof(ModelSmall::Smem);
        if (in_f64) pdl(k_build_models<true, ModelSmall, 256>, count, 256, sm, st, segs, idx, src, models, cfg);
        else pdl(k_build_models<false, ModelSmall, 256>, count, 256, sm, st, segs, idx, src, models, cfg);
    }
}

void launch_first_sample(const SegDesc* seg, const void* src, int in_f64, uint8_t* models, const DevCfg& cfg,
                         uint8_t* aux, uint32_t aux_budget, uint32_t* gate, cudaStream_t st, const uint64_t* pre,
                         uint32_t* dslices) {
    size_t sm = sizeof(ModelMid::Smem);
    if (in_f64) pdl(k_first_sample<true>, 1, 512, sm, st, pre, seg, src, models, cfg, aux, aux_budget, gate, dslices);
    else pdl(k_first_sample<false>, 1, 512, sm, st, pre, seg, src, models, cfg, aux, aux_budget, gate, dslices);
}

void launch_gather(const SegDesc* seg, const void* src, int in_f64, uint64_t seed, uint64_t j0, uint64_t s,
                   uint64_t* out, const uint32_t* gate, cudaStream_t st) {
    int grid = (int)std::min<uint64_t>((s + 255) / 256, (uint64_t)num_sms() * 8);
    if (grid < 1) grid = 1;
    if (in_f64) pdl(k_gather<true>, grid, 256, 0, st, seg, src, seed, j0, s, out, gate);
    else pdl(k_gather<false>, grid, 256, 0, st, seg, src, seed, j0, s, out, gate);
}

void launch_train_rmi(const uint64_t* sample, uint64_t s, uint32_t B, uint8_t* model, uint32_t nbuckets, void* ws,
                      const uint32_t* gate, cudaStream_t st) {
    const uint32_t n = (uint32_t)s;
    const uint32_t nch = (uint32_t)((s + kTrainChunk - 1) / kTrainChunk);
    RmiEntry* E = (RmiEntry*)(model + sizeof(ModelHdr));
    static_assert(kBigSplit == kBigSplitWS, "workspace layout");
    // (before the kernel chain: a memset between two programmatic-launch
    // kernels serialises them fully; no kernel before k_train_bigfits uses it)
    cudaMemsetAsync(train_ws(ws, s, B).bigcnt, 0, 4 * (size_t)B, st);
    pdl(k_train_sums<false>, nch, kTrainNT, 0, st, sample, n, ws, B, gate);
    pdl(k_train_reduce<false>, 1, kTrainNT, 0, st, sample, n, ws, B, gate);
    pdl(k_train_sums<true>, nch, kTrainNT, 0, st, sample, n, ws, B, gate);
    pdl(k_train_reduce<true>, 1, kTrainNT, 0, st, sample, n, ws, B, gate);
    const int gb = (int)std::min<uint64_t>((s + kTrainNT - 1) / kTrainNT, (uint64_t)num_sms() * 8);
    pdl(k_train_bounds, gb, kTrainNT, 0, st, sample, n, ws, B, gate);
    pdl(k_train_fits, (B + kFitWarps - 1) / kFitWarps, 32 * kFitWarps, 0, st, sample, n, ws, B, E, gate);
    const int gbig = (int)std::min<uint64_t>((uint64_t)B * kBigSplit, (uint64_t)num_sms() * 4);
    pdl(k_train_bigfits, gbig, kBigFitNT, 0, st, sample, n, ws, B, E, gate);
    pdl(k_train_enforce, 1, kEnforceNT, 16 * (size_t)B, st, sample, n, ws, B, model, nbuckets, gate);
}

void launch_tree_build(const uint64_t* sorted, uint64_t s, uint32_t budget, int eq_mode, uint8_t* model,
                       cudaStream_t st) {
    pdl(k_tree_build, 1, 512, sizeof(ModelMid::Smem), st, sorted, (uint32_t)s, budget, eq_mode, model);
}

void launch_block_sort(uint64_t* keys, uint64_t n, cudaStream_t st) {
    pdl(k_block_sort, 1, 512, sizeof(ModelMid::Smem), st, keys, (uint32_t)n);
}

}  // namespace lsort_dev
