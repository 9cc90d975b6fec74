// cluster.cu -- the last distribution level fused with the base case, in
// distributed shared memory (thread-block clusters, sm_90+ / sm_100a).
//
// A segment of up to kClCap keys (a level-0 bucket of ~1e5 keys at the
// BASELINE sizes) is owned by one cluster of kClSize CTAs:
//   1. every CTA streams its 1/kClSize share of the segment: min / max,
//      combined across the cluster through DSMEM;
//   2. sub-bucket = (key - min) >> shift, S = 2^k sub-buckets of ~1.5-3 K
//      keys (the learned level above has made the segment's keys locally
//      uniform, so equal-width sub-ranges are balanced -- and need no model);
//   3. per-CTA histograms are exchanged through DSMEM; sub-buckets are
//      assigned in order to owner CTAs (contiguous ranges, balanced);
//   4. each CTA re-streams its share (L2-resident) and stores every key
//      straight into its owner's shared memory (st.shared::cluster);
//   5. each CTA sorts its sub-buckets in shared memory (SmemSort first pass
//      with keys in registers) and writes them to their final position,
//      decoding float keys on the way out.
// One HBM read and one HBM write per key replace the classify + scatter of
// a further level plus the base-case pass.
// Sub-buckets too large for one CTA (skewed segments) are written to the
// level's output buffer and queued as base-case / recursion work items.
#include <cooperative_groups.h>

#include <algorithm>

#include "kernels_common.cuh"
#include "smemsort.cuh"

namespace cg = cooperative_groups;

namespace lsort_dev {

using ClSS = SmemSort<kClNT, kClSortCap, kClSortCap>;
static_assert(kClCap / kClTarget <= (uint32_t)kClSub, "sub-bucket table too small");

struct ClSmem {
    uint64_t recv[kClRecv];         // keys received from the cluster (owned sub-buckets)
    ClSS::SmemR ss;                 // sub-bucket sort workspace
    uint32_t cnt[kClSub];           // this CTA's share: keys per sub-bucket (read remotely)
    uint32_t pre[kClSub];           // keys of lower-ranked CTAs per sub-bucket
    uint32_t cur[kClSub];           // send cursors
    uint32_t dsl[kClSub];           // owner << 24 | offset in owner's recv, ~0 = global
    uint32_t start[kClSub + 1];     // sub-bucket start within the segment
    uint64_t mm[2];                 // this CTA's min / max (read remotely)
    uint64_t red[2 * (kClNT / 32)];
    uint64_t gmm[2];
    uint4 bat[kClSub];              // sort batches: first / end sub-bucket, keys, digits
    uint32_t nbat;
};

template <bool OUT_F64>
__global__ void __cluster_dims__(kClSize, 1, 1) __launch_bounds__(kClNT, 1)
    k_cluster_sort(const BaseItem* segs, uint32_t nsegs, const uint64_t* src, uint64_t* dst, void* out,
                   LevelParams p, uint32_t depth) {
    extern __shared__ uint4 smem_u4[];
    ClSmem& M = *(ClSmem*)smem_u4;
    cg::cluster_group cl = cg::this_cluster();
    const uint32_t rank = cl.block_rank();
    const uint32_t cid = blockIdx.x / kClSize, ncl = gridDim.x / kClSize;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (p.ctrl->nan_index != ~0ull) return;  // uniform across the grid
    for (uint32_t si = cid; si < nsegs; si += ncl) {
        const BaseItem sg = segs[si];
        const uint32_t n = (uint32_t)sg.n;
        const uint64_t* g = src + sg.begin;
        const uint32_t lo = (uint32_t)((uint64_t)n * rank / kClSize);
        const uint32_t hi = (uint32_t)((uint64_t)n * (rank + 1) / kClSize);
        // ---- 1. min / max over the cluster
        uint64_t mn = ~0ull, mx = 0;
        for (uint32_t i = lo + tid; i < hi; i += kClNT) {
            const uint64_t k = g[i];
            mn = k < mn ? k : mn;
            mx = k > mx ? k : mx;
        }
        mn = block_reduce_min<kClNT>(mn, M.red);
        mx = block_reduce_max<kClNT>(mx, M.red);
        if (tid == 0) { M.mm[0] = mn; M.mm[1] = mx; }
        cl.sync();
        if (warp == 0) {
            uint64_t a = ~0ull, b = 0;
            if (lane < kClSize) {
                const uint64_t* r = cl.map_shared_rank(M.mm, lane);
                a = r[0];
                b = r[1];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t a2 = __shfl_xor_sync(FULL_MASK, a, o), b2 = __shfl_xor_sync(FULL_MASK, b, o);
                a = a2 < a ? a2 : a;
                b = b2 > b ? b2 : b;
            }
            if (lane == 0) { M.gmm[0] = a; M.gmm[1] = b; }
        }
        __syncthreads();
        mn = M.gmm[0];
        mx = M.gmm[1];
        if (mn == mx) {  // homogeneous segment: value stores only
            for (uint32_t i = lo + tid; i < hi; i += kClNT) {
                if (OUT_F64) ((double*)out)[sg.begin + i] = decode(mn);
                else ((uint64_t*)out)[sg.begin + i] = mn;
            }
            if (rank == 0 && tid == 0) atomicAdd(&p.ctrl->keys_fill, (unsigned long long)n);
            cl.sync();  // remote reads of M.mm are done before the next segment
            continue;
        }
        // ---- 2. sub-buckets: equal-width ranges, 1.5-3 K keys each on average
        uint32_t lgs = 1;
        while ((1u << lgs) < kClSub && ((uint64_t)kClTarget << lgs) < n) ++lgs;
        const uint32_t S = 1u << lgs;
        const uint32_t bits = bitlen64(mx - mn);
        const uint32_t shift = bits > lgs ? bits - lgs : 0;
        for (uint32_t b = tid; b < S; b += kClNT) { M.cnt[b] = 0; M.cur[b] = 0; }
        __syncthreads();
        for (uint32_t i = lo + tid; i < hi; i += kClNT) atomicAdd(&M.cnt[(uint32_t)((g[i] - mn) >> shift)], 1u);
        cl.sync();
        // ---- 3. exchange counts, place sub-buckets
        for (uint32_t b = tid; b < S; b += kClNT) {
            uint32_t tot = 0, pre = 0;
#pragma unroll
            for (int q = 0; q < kClSize; ++q) {
                const uint32_t c = cl.map_shared_rank(M.cnt, q)[b];
                pre += (uint32_t)q < rank ? c : 0u;
                tot += c;
            }
            M.pre[b] = pre;
            M.start[b] = tot;
        }
        __syncthreads();
        if (tid == 0) {  // sequential placement (S <= kClSub); identical in every CTA
            // owner = the CTA whose 1/kClSize slice of the segment holds the
            // sub-bucket's midpoint: load <= target + kClSortCap <= kClRecv
            const uint32_t target = (n + kClSize - 1) / kClSize;
            uint32_t run = 0, cur_owner = 0, load = 0;
            for (uint32_t b = 0; b < S; ++b) {
                const uint32_t t = M.start[b];
                M.start[b] = run;
                uint32_t d = ~0u;
                if (t <= (uint32_t)kClSortCap) {
                    const uint32_t owner = min((uint32_t)kClSize - 1, (run + t / 2) / target);
                    if (owner != cur_owner) { cur_owner = owner; load = 0; }
                    if (load + t <= (uint32_t)kClRecv) { d = owner << 24 | load; load += t; }
                }
                M.dsl[b] = d;
                run += t;
            }
            M.start[S] = run;
        }
        __syncthreads();
        // sub-buckets that stay in global memory become work items (rank 0 queues them)
        if (rank == 0) {
            for (uint32_t b = tid; b < S; b += kClNT) {
                const uint32_t len = M.start[b + 1] - M.start[b];
                if (M.dsl[b] != ~0u || len == 0) continue;
                const uint64_t begin = sg.begin + M.start[b];
                if (len <= p.base_cap[2]) {
                    const int c = len <= p.base_cap[0] ? 0 : (len <= p.base_cap[1] ? 1 : 2);
                    const unsigned e = atomicAdd(&p.ctrl->n_base[c], 1u);
                    if (e < p.list_cap) p.base[c][e] = BaseItem{begin, len, (int64_t)begin};
                    else atomicOr(&p.ctrl->err, 2u);
                    atomicAdd(&p.ctrl->keys_base, (unsigned long long)len);
                } else {
                    const unsigned e = atomicAdd(&p.ctrl->n_rec, 1u);
                    if (e < p.list_cap) p.rec[e] = SegOut{begin, len, depth, depth > p.depth_cap ? kSegForceRadix : 0u, 0, begin};
                    else atomicOr(&p.ctrl->err, 4u);
                    atomicAdd(&p.ctrl->keys_rec, (unsigned long long)len);
                }
            }
        }
        // ---- 4. send every key of the share to its owner (or to global)
        for (uint32_t i = lo + tid; i < hi; i += kClNT) {
            const uint64_t k = g[i];
            const uint32_t b = (uint32_t)((k - mn) >> shift);
            const uint32_t r = atomicAdd(&M.cur[b], 1u) + M.pre[b];
            const uint32_t d = M.dsl[b];
            if (d != ~0u) cl.map_shared_rank(M.recv, d >> 24)[(d & 0xffffffu) + r] = k;
            else dst[sg.begin + M.start[b] + r] = k;
        }
        cl.sync();  // all keys delivered (release / acquire across the cluster)
        // ---- 5. sort owned sub-buckets in batches of <= kClSortCap keys:
        // one counting pass per batch, digit = batch base of the sub-bucket +
        // the next lg(len) bits below the sub-bucket bits (monotone in the key)
        uint32_t* dbase = M.cur;  // free after the send
        uint32_t* lgd = M.cnt;    // free after the exchange (remote reads ended at the last cluster barrier)
        if (tid == 0) {
            uint32_t nbat = 0, b = 0;
            while (b < S) {
                const uint32_t d0 = M.dsl[b];
                if (d0 == ~0u || (d0 >> 24) != rank || M.start[b + 1] == M.start[b]) { ++b; continue; }
                const uint32_t b0 = b;
                uint32_t tot = 0, nd = 0;
                while (b < S) {
                    const uint32_t d = M.dsl[b];
                    const uint32_t len = M.start[b + 1] - M.start[b];
                    const uint32_t lg = len > 1 ? min(31u - __clz(len), shift) : 0u;  // pow2 floor digits
                    // (an empty sub-bucket still takes one digit: the digits are bounded like the keys)
                    if (d == ~0u || (d >> 24) != rank || tot + len > (uint32_t)kClSortCap ||
                        nd + (1u << lg) > (uint32_t)kClSortCap)
                        break;
                    dbase[b] = nd;
                    lgd[b] = lg;
                    nd += 1u << lg;
                    tot += len;
                    ++b;
                }
                M.bat[nbat++] = make_uint4(b0, b, tot, nd);
            }
            M.nbat = nbat;
        }
        __syncthreads();
        const uint32_t nbat = M.nbat;
        for (uint32_t q = 0; q < nbat; ++q) {
            const uint4 bt = M.bat[q];
            const uint32_t b0 = bt.x, tot = bt.z, nd = bt.w;
            const uint32_t off = M.dsl[b0] & 0xffffffu;
            const uint64_t ob = sg.begin + M.start[b0];
            uint64_t k[ClSS::ITEMS];
            uint32_t dg[ClSS::ITEMS];
#pragma unroll
            for (int i = 0; i < ClSS::ITEMS; ++i) {
                const uint32_t j = tid + i * kClNT;
                k[i] = j < tot ? M.recv[off + j] : mn;
                const uint64_t x = k[i] - mn;
                const uint32_t sb = (uint32_t)(x >> shift);
                const uint32_t lg = j < tot ? lgd[sb] : 0u;
                dg[i] = j < tot ? dbase[sb] + (uint32_t)((x >> (shift - lg)) & ((1ull << lg) - 1ull)) : 0u;
            }
            if (off + tot > (uint32_t)kClRecv || nd > (uint32_t)kClSortCap) {  // cannot happen: placement invariant
                atomicOr(&p.ctrl->err, 64u);
                continue;
            }
            ClSS::sort_digits(k, dg, tot, nd, M.ss, dst + ob);
            for (uint32_t i = tid; i < tot; i += kClNT) {
                const uint64_t v = M.ss.B[i];
                if (OUT_F64) __stcs((double*)out + ob + i, decode(v));
                else __stcs((unsigned long long*)out + ob + i, (unsigned long long)v);
            }
            if (tid == 0) atomicAdd(&p.ctrl->keys_base, (unsigned long long)tot);
            __syncthreads();
        }
        cl.sync();  // shared memory of every CTA may be reused for the next segment
    }
}

static int g_cluster_grid = -1;

void cluster_init(int optin) {
    (void)optin;
    const size_t sm = sizeof(ClSmem);
    if (cudaFuncSetAttribute(k_cluster_sort<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess ||
        cudaFuncSetAttribute(k_cluster_sort<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) !=
            cudaSuccess) {
        cudaGetLastError();
        g_cluster_grid = 0;
        return;
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(kClSize * 64, 1, 1);
    lc.blockDim = dim3(kClNT, 1, 1);
    lc.dynamicSmemBytes = sm;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = kClSize;
    at.val.clusterDim.y = 1;
    at.val.clusterDim.z = 1;
    lc.attrs = &at;
    lc.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, (void*)k_cluster_sort<true>, &lc) != cudaSuccess) {
        cudaGetLastError();
        ncl = 0;
    }
    g_cluster_grid = ncl * kClSize;
}

bool cluster_available() { return g_cluster_grid > 0; }

void launch_cluster_sort(const BaseItem* segs, uint32_t nsegs, const uint64_t* src, uint64_t* dst, void* out,
                         int out_f64, const LevelParams& p, uint32_t depth, cudaStream_t st) {
    if (!nsegs) return;
    const int grid = std::min<int>(g_cluster_grid, (int)nsegs * kClSize);
    const size_t sm = sizeof(ClSmem);
    if (out_f64) k_cluster_sort<true><<<grid, kClNT, sm, st>>>(segs, nsegs, src, dst, out, p, depth);
    else k_cluster_sort<false><<<grid, kClNT, sm, st>>>(segs, nsegs, src, dst, out, p, depth);
}

}  // namespace lsort_dev
