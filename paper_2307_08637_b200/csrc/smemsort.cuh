// smemsort.cuh -- shared-memory segment sort (GPU base case and model
// sample sort). See SmemSort below.
#pragma once

#include "kernels_common.cuh"

namespace lsort_dev {

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
    // (inlined: as an out-of-line call the shared-memory accesses through `S`
    // become generic loads/stores)
    __device__ static __forceinline__ void pass(uint64_t* a, uint64_t* b, uint32_t off, uint32_t len, Smem& S) {
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

    __device__ static __forceinline__ void warp_rank_sort(uint64_t* a, uint32_t len) {
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

}  // namespace lsort_dev
