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
    static_assert(NBMAX <= 65536, "digit indices are kept in 16 bits");
    static constexpr int kSmall = 16;
    static constexpr int kMedium = 256;
    static constexpr int kStk = CAP / (kSmall + 1) + 2;
    static_assert(CAP < 65536, "16-bit offsets, lengths and ranks");
    struct Smem {
        uint64_t A[CAP + 4];  // logical key i at A[mis + i]
        uint64_t B[CAP];
        uint32_t hist[NBMAX + 1];
        uint16_t R[CAP];
        uint32_t wsum[NT / 32 + 1];
        uint64_t red[2 * (NT / 32)];
        uint32_t n_med, n_large, n_l4, n_l16;
        uint16_t med_off[kStk], med_len[kStk], large_off[kStk], large_len[kStk];
        uint64_t mbar;
    };
    // the same without the input array A (keys arrive in registers; scratch
    // for the rare large-digit passes is supplied by the caller)
    struct SmemR {
        uint64_t B[CAP];
        uint32_t hist[NBMAX + 1];
        uint16_t R[CAP / 2];  // collision-digit lists only (<= n / 2 digits hold >= 2 keys)
        uint32_t wsum[NT / 32 + 1];
        uint64_t red[2 * (NT / 32)];
        uint32_t n_med, n_large, n_l4, n_l16;
        uint16_t med_off[kStk], med_len[kStk], large_off[kStk], large_len[kStk];
    };

    template <class SM>
    __device__ static __forceinline__ void push(SM& S, uint32_t at, uint32_t l) {
        if (l <= (uint32_t)kMedium) {
            uint32_t q = atomicAdd(&S.n_med, 1u);
            S.med_off[q] = (uint16_t)at;
            S.med_len[q] = (uint16_t)l;
        } else {
            uint32_t q = atomicAdd(&S.n_large, 1u);
            S.large_off[q] = (uint16_t)at;
            S.large_len[q] = (uint16_t)l;
        }
    }

    // one distribution pass over a[off, off+len), staging through b
    // (inlined: as an out-of-line call the shared-memory accesses through `S`
    // become generic loads/stores)
    template <class SM>
    __device__ static __forceinline__ void pass(uint64_t* a, uint64_t* b, uint32_t off, uint32_t len, SM& S) {
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
        for (uint32_t i = tid; i < len; i += NT) atomicAdd(&S.hist[(uint32_t)((a[off + i] - mn) >> shift)], 1u);
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
        }
        __syncthreads();
        // placement by atomic cursors (order inside a digit is arbitrary: the
        // fix-up below ranks each key among its digit); afterwards hist[d] holds
        // the END of digit d, i.e. the start of digit d + 1
        for (uint32_t i = tid; i < len; i += NT) {
            const uint64_t k = a[off + i];
            b[off + atomicAdd(&S.hist[(uint32_t)((k - mn) >> shift)], 1u)] = k;
        }
        __syncthreads();
        for (uint32_t j = tid; j < len; j += NT) {
            const uint64_t k = b[off + j];
            const uint32_t d = (uint32_t)((k - mn) >> shift);
            const uint32_t s0 = d ? S.hist[d - 1] : 0u, c = S.hist[d] - s0;
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

    // rank sort of a[0,len) by one warp, Q keys per lane (len <= 32 * Q)
    template <int Q>
    __device__ static __forceinline__ void warp_rank_sort_q(uint64_t* a, uint32_t len) {
        const int lane = threadIdx.x & 31;
        uint64_t v[Q];
        uint32_t r[Q];
        uint64_t mn = ~0ull, mx = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint32_t idx = lane + 32 * q;
            v[q] = idx < len ? a[idx] : ~0ull;
            r[q] = 0;
            if (idx < len) {
                mn = v[q] < mn ? v[q] : mn;
                mx = v[q] > mx ? v[q] : mx;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t a1 = __shfl_xor_sync(FULL_MASK, mn, o), b1 = __shfl_xor_sync(FULL_MASK, mx, o);
            mn = a1 < mn ? a1 : mn;
            mx = b1 > mx ? b1 : mx;
        }
        if (mn == mx) return;  // all equal (duplicate-heavy digit): already sorted
        for (uint32_t j = 0; j < len; ++j) {
            const uint64_t w = a[j];
#pragma unroll
            for (int q = 0; q < Q; ++q) r[q] += (w < v[q]) || (w == v[q] && j < (uint32_t)(lane + 32 * q));
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if ((uint32_t)(lane + 32 * q) < len) a[r[q]] = v[q];
        __syncwarp();
    }
    __device__ static __forceinline__ void warp_rank_sort(uint64_t* a, uint32_t len) {
        if (len <= 32) warp_rank_sort_q<1>(a, len);
        else if (len <= 64) warp_rank_sort_q<2>(a, len);
        else if (len <= 128) warp_rank_sort_q<4>(a, len);
        else warp_rank_sort_q<8>(a, len);
    }

    // Sort the pushed medium / large digit ranges of arr (scratch: same size).
    template <class SM>
    __device__ static void drain(uint64_t* arr, uint64_t* scratch, SM& S) {
        const int warp = threadIdx.x >> 5;
        for (;;) {
            const uint32_t nm = S.n_med, nl = S.n_large;
            if (nm == 0 && nl == 0) break;
            for (uint32_t e = warp; e < nm; e += NT / 32) warp_rank_sort(arr + S.med_off[e], S.med_len[e]);
            __syncthreads();
            if (threadIdx.x == 0) S.n_med = 0;
            if (nl == 0) { __syncthreads(); break; }
            const uint32_t off = S.large_off[nl - 1], len = S.large_len[nl - 1];
            __syncthreads();
            if (threadIdx.x == 0) S.n_large = nl - 1;
            pass(arr, scratch, off, len, S);
            __syncthreads();
        }
    }

    // sort a[0,n) (keys already in shared memory)
    __device__ static void sort(uint64_t* a, uint32_t n, Smem& S) {
        if (threadIdx.x == 0) { S.n_med = 0; S.n_large = 0; }
        __syncthreads();
        pass(a, S.B, 0, n, S);
        __syncthreads();
        drain(a, S.B, S);
    }

    __device__ static __forceinline__ void cswap(uint64_t& a, uint64_t& b) {
        const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
        a = lo;
        b = hi;
    }

    // Register-resident first pass (ITEMS = CAP / NT keys per thread, read once
    // from a): min/max, one counting pass with >= 1 digit per key, placement
    // into S.B, in-place rank fix of digits with 2..kSmall keys. Then the
    // remaining digits are drained with S.A as scratch. Result in S.B.
    // (a may alias S.A: it is not read after the first pass.)
    static constexpr int ITEMS = CAP / NT;
    static constexpr int kThreads = NT;
    static constexpr uint32_t kNbMax = CAP < NBMAX ? CAP : NBMAX;  // digits of one counting pass
    __device__ static void sort_fast(const uint64_t* a, uint32_t n, Smem& S, bool eq = false) {
        static_assert(ITEMS * NT == CAP, "CAP must be a multiple of NT");
        uint64_t k[ITEMS];
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const uint32_t j = threadIdx.x + i * NT;
            k[i] = j < n ? a[j] : 0ull;
        }
        sort_regs(k, n, S, S.A, eq);
    }
    // keys j = threadIdx.x + i * NT in k[i]; result in S.B; scratch: >= n keys
    template <int IT = ITEMS, class SM>
    // eq: equalised digits for skewed key sets spanning a wide range (a root's
    // sample: encoded floats crowd into a few binades -- Normal's first sample put
    // 77% of its keys into digits of > 256 keys, drained one digit at a time):
    // a coarse histogram of the top 10 digit bits, and each key's digit
    // interpolated inside its coarse bin by its key offset -- monotone, ~1 key
    // per digit for any smooth distribution.
    __device__ static void sort_regs(uint64_t (&k)[IT], uint32_t n, SM& S, uint64_t* scratch, bool eq = false) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        constexpr int NW = NT / 32;
        constexpr uint32_t kNb = CAP < NBMAX ? CAP : NBMAX;  // digits: >= 1 per key for n near CAP
        // nb = smallest power of two >= n (capped): <= 1 key per digit on average
        const uint32_t lgnb = min(32u - __clz(max(n, 2u) - 1u), 31u - __clz(kNb));
        const uint32_t nb = 1u << lgnb;
        // digit = (key - base) >> shift, monotone and < nb. base / shift come
        // from 32-bit reductions: the range of the high words, and when every
        // key shares one high word, the range of the low words; only a high
        // range of 1..7 words (keys straddling a 2^32 boundary) needs the
        // exact 64-bit min / max.
        uint32_t* redh = (uint32_t*)S.red;  // 2 * NW words (S.red holds 2 * NW u64)
        auto reduce32 = [&](uint32_t lo, uint32_t hi, uint32_t& mn, uint32_t& mx) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo = min(lo, __shfl_xor_sync(FULL_MASK, lo, o));
                hi = max(hi, __shfl_xor_sync(FULL_MASK, hi, o));
            }
            if (lane == 0) { redh[2 * warp] = lo; redh[2 * warp + 1] = hi; }
            __syncthreads();
            uint32_t a1 = lane < NW ? redh[2 * lane] : ~0u, b1 = lane < NW ? redh[2 * lane + 1] : 0u;
#pragma unroll
            for (int o = NW / 2; o > 0; o >>= 1) {
                a1 = min(a1, __shfl_xor_sync(FULL_MASK, a1, o));
                b1 = max(b1, __shfl_xor_sync(FULL_MASK, b1, o));
            }
            mn = __shfl_sync(FULL_MASK, a1, 0);
            mx = __shfl_sync(FULL_MASK, b1, 0);
            // (no trailing barrier: the next writer of redh / S.red syncs first)
        };
        // the digit histogram is zeroed here, before the first barrier, instead
        // of behind a barrier of its own in sort_digits
        {
            const uint32_t nbz = (nb + 3) & ~3u;
            for (uint32_t d = tid; d < nbz; d += NT) S.hist[d] = 0;
        }
        uint32_t mnh, mxh;
        {
            uint32_t lo = ~0u, hi = 0;
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint32_t j = tid + i * NT;
                const uint32_t h = (uint32_t)(k[i] >> 32);
                if (j < n) { lo = min(lo, h); hi = max(hi, h); }
            }
            reduce32(lo, hi, mnh, mxh);
        }
        const uint32_t dh = mxh - mnh;
        uint64_t base = (uint64_t)mnh << 32;
        uint32_t shift;
        if (dh >= 8) {
            // window [mnh << 32, (mxh + 1) << 32) of 2^(32 + bits) keys; the
            // true span is at least (dh - 1) << 32, >= 7/16 of it
            shift = 32u + (32u - __clz(dh)) - lgnb;
        } else if (dh == 0) {
            uint32_t lo = ~0u, hi = 0, mnl, mxl;
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint32_t j = tid + i * NT;
                if (j < n) { lo = min(lo, (uint32_t)k[i]); hi = max(hi, (uint32_t)k[i]); }
            }
            __syncthreads();  // redh of the high-word reduction is read
            reduce32(lo, hi, mnl, mxl);
            if (mnl == mxl) {  // homogeneous: already sorted
#pragma unroll
                for (int i = 0; i < IT; ++i) {
                    const uint32_t j = tid + i * NT;
                    if (j < n) S.B[j] = k[i];
                }
                __syncthreads();
                return;
            }
            const uint32_t bits = 32u - __clz(mxl - mnl);
            base |= mnl;
            shift = bits > lgnb ? bits - lgnb : 0;
        } else {  // keys straddle 1..7 high-word boundaries: exact 64-bit range
            uint64_t mn = ~0ull, mx = 0;
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint32_t j = tid + i * NT;
                if (j < n) {
                    mn = k[i] < mn ? k[i] : mn;
                    mx = k[i] > mx ? k[i] : mx;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t a1 = __shfl_xor_sync(FULL_MASK, mn, o), b1 = __shfl_xor_sync(FULL_MASK, mx, o);
                mn = a1 < mn ? a1 : mn;
                mx = b1 > mx ? b1 : mx;
            }
            __syncthreads();  // redh of the high-word reduction is read
            if (lane == 0) { S.red[2 * warp] = mn; S.red[2 * warp + 1] = mx; }
            __syncthreads();
            uint64_t a1 = lane < NW ? S.red[2 * lane] : ~0ull, b1 = lane < NW ? S.red[2 * lane + 1] : 0ull;
#pragma unroll
            for (int o = NW / 2; o > 0; o >>= 1) {
                const uint64_t a2 = __shfl_xor_sync(FULL_MASK, a1, o), b2 = __shfl_xor_sync(FULL_MASK, b1, o);
                a1 = a2 < a1 ? a2 : a1;
                b1 = b2 > b1 ? b2 : b1;
            }
            mn = __shfl_sync(FULL_MASK, a1, 0);
            mx = __shfl_sync(FULL_MASK, b1, 0);
            __syncthreads();  // S.red is reused by the scan
            const uint32_t bits = bitlen64(mx - mn);  // mx > mn: the high words differ
            base = mn;
            shift = bits > lgnb ? bits - lgnb : 0;
        }
        uint32_t dg[IT];
        if (eq && lgnb >= 10 && NBMAX >= 1024) {
            const uint32_t cs = shift + lgnb - 10;  // coarse bin: top 10 bits of the digit
            // S.hist[0, nb) is zero (zeroed before the range reduction's barrier)
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint32_t j = tid + i * NT;
                if (j < n) atomicAdd(&S.hist[(uint32_t)((k[i] - base) >> cs)], 1u);
            }
            __syncthreads();
            block_exclusive_scan_u32<NT>(S.hist, 1024, S.wsum);
            if (tid == 0) S.hist[1024] = n;
            __syncthreads();
            const double scale = (double)nb / (double)n, unit = ldexp(1.0, -(int)cs);
#pragma unroll
            for (int i = 0; i < IT; ++i) {
                const uint64_t off = k[i] - base;
                const uint32_t bin = (uint32_t)(off >> cs);
                const uint32_t c0 = S.hist[min(bin, 1023u)], c1 = S.hist[min(bin, 1023u) + 1];
                const double t = (double)(off - ((uint64_t)bin << cs)) * unit;  // [0, 1]
                const double f = (double)c0 + t * (double)(c1 - c0);
                dg[i] = min((uint32_t)(f * scale), nb - 1);
            }
            __syncthreads();  // coarse counts read: the counting pass re-zeroes hist
            sort_digits<IT, SM, false>(k, dg, n, nb, S, scratch);
            return;
        }
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            dg[i] = (uint32_t)((k[i] - base) >> shift);
        }
        // shift 0: a digit is one key value -- keys sharing a digit are equal and need
        // no fix-up (duplicate-heavy small-range integer segments)
        sort_digits<IT, SM, true>(k, dg, n, nb, S, scratch, shift == 0);
    }

    // Counting pass on caller-supplied digits (dg[i] < nb <= NBMAX, monotone in
    // the key), placement into S.B, collision fix-up, drain of large digits.
    // Result in S.B. The caller has zeroed nothing; S.n_* are reset here.
    // ZEROED: the caller zeroed hist[0, roundup4(nb)) before a barrier it has passed
    template <int IT = ITEMS, class SM, bool ZEROED = false>
    __device__ static void sort_digits(uint64_t (&k)[IT], const uint32_t (&dg)[IT], uint32_t n, uint32_t nb,
                                       SM& S, uint64_t* scratch, bool exact = false) {
        const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
        uint64_t* B = S.B;
        nb = (nb + 3) & ~3u;  // whole 16-byte groups for the vectorised scan (extra digits stay empty)
        if (tid == 0) { S.n_med = 0; S.n_large = 0; S.n_l4 = 0; S.n_l16 = 0; }
        if (!ZEROED) {
            for (uint32_t d = tid; d < nb; d += NT) S.hist[d] = 0;
            __syncthreads();
        }
        uint32_t dp[IT];  // digit << 16 | rank within the digit
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const uint32_t j = tid + i * NT;
            dp[i] = j < n ? (dg[i] << 16 | atomicAdd(&S.hist[dg[i]], 1u)) : 0u;
        }
        __syncthreads();
        // exclusive scan of the digit counts, fused with the compaction of the
        // collision digits: one packed 64-bit scan carries (keys | digits with
        // 2..4 keys << 16 | digits with 5..kSmall keys << 32), so every thread
        // knows where its collision digits go in the two lists (S.R front /
        // back) without atomics or a second pass over the digits
        uint32_t n4, n16;
        constexpr uint32_t kR = sizeof(S.R) / sizeof(S.R[0]);  // list capacity (front: 2..4 keys, back: 5..kSmall)
        {
            static_assert(CAP < 65536, "packed 16-bit scan fields");
            const uint32_t per = (nb + NT - 1) / NT;
            const uint32_t lo = min(nb, tid * per), hi = min(nb, lo + per);
            auto pk = [](uint32_t h) -> uint64_t {  // (h-2) <= 2 <=> 2..4; (h-5) <= kSmall-5 <=> 5..kSmall
                return (uint64_t)h | ((uint64_t)(h - 2u <= 2u) << 16) |
                       ((uint64_t)(h - 5u <= (uint32_t)kSmall - 5u) << 32);
            };
            uint64_t sum = 0;
            if (per % 4 == 0) {  // 16-byte reads: no bank conflicts between the threads' chunks
                for (uint32_t d = lo; d < hi; d += 4) {
                    const uint4 h4 = *(const uint4*)&S.hist[d];
                    sum += pk(h4.x) + pk(h4.y) + pk(h4.z) + pk(h4.w);
                }
            } else {
                for (uint32_t d = lo; d < hi; ++d) sum += pk(S.hist[d]);
            }
            uint64_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t w = __shfl_up_sync(FULL_MASK, incl, o);
                if (lane >= o) incl += w;
            }
            if (lane == 31) S.red[warp] = incl;
            __syncthreads();
            constexpr int NW = NT / 32;
            uint64_t wv = lane < NW ? S.red[lane] : 0ull, wincl = wv;
#pragma unroll
            for (int o = 1; o < NW; o <<= 1) {
                const uint64_t w = __shfl_up_sync(FULL_MASK, wincl, o);
                if (lane >= o) wincl += w;
            }
            const uint64_t total = __shfl_sync(FULL_MASK, wincl, NW - 1);
            n4 = (uint32_t)(total >> 16) & 0xffffu;
            n16 = (uint32_t)(total >> 32) & 0xffffu;
            const uint64_t ex = incl - sum + __shfl_sync(FULL_MASK, wincl - wv, warp);
            uint32_t run = (uint32_t)ex & 0xffffu, p4 = (uint32_t)(ex >> 16) & 0xffffu,
                     p16 = (uint32_t)(ex >> 32) & 0xffffu;
            auto place = [&](uint32_t d, uint32_t h, uint32_t at) {
                if (h < 2 || exact) return;  // the common case: empty / single-key digit (exact: all equal)
                if (h <= 4) S.R[p4++] = (uint16_t)d;  // digit index (< NBMAX <= 65536)
                else if (h <= (uint32_t)kSmall) S.R[kR - 1 - (p16++)] = (uint16_t)d;
                else push(S, at, h);
            };
            if (per % 4 == 0) {
                for (uint32_t d = lo; d < hi; d += 4) {
                    const uint4 h4 = *(const uint4*)&S.hist[d];
                    uint4 o4;
                    o4.x = run; run += h4.x;
                    o4.y = run; run += h4.y;
                    o4.z = run; run += h4.z;
                    o4.w = run; run += h4.w;
                    *(uint4*)&S.hist[d] = o4;
                    place(d, h4.x, o4.x);
                    place(d + 1, h4.y, o4.y);
                    place(d + 2, h4.z, o4.z);
                    place(d + 3, h4.w, o4.w);
                }
            } else {
                for (uint32_t d = lo; d < hi; ++d) {
                    const uint32_t t = S.hist[d];
                    S.hist[d] = run;
                    place(d, t, run);
                    run += t;
                }
            }
            if (tid == 0) S.hist[nb] = n;
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < IT; ++i) {
            const uint32_t j = tid + i * NT;
            if (j < n) {
                B[S.hist[dp[i] >> 16] + (dp[i] & 0xffffu)] = k[i];
            }
        }
        __syncthreads();
        // collision digits: 2..4 keys by a fixed 4-key network (pad ~0),
        // 5..kSmall keys by insertion sort (rare); all lanes on list entries
        if (exact) n4 = n16 = 0;  // (CTA-uniform) equal keys: nothing to fix
        for (uint32_t e = tid; e < n4; e += NT) {
            const uint32_t d = S.R[e], s0 = S.hist[d], c = S.hist[d + 1] - s0;
            uint64_t x0 = B[s0], x1 = B[s0 + 1];
            uint64_t x2 = c >= 3 ? B[s0 + 2] : ~0ull, x3 = c == 4 ? B[s0 + 3] : ~0ull;
            cswap(x0, x1); cswap(x2, x3); cswap(x0, x2); cswap(x1, x3); cswap(x1, x2);
            B[s0] = x0;
            B[s0 + 1] = x1;
            if (c >= 3) B[s0 + 2] = x2;
            if (c == 4) B[s0 + 3] = x3;
        }
        for (uint32_t e = tid; e < n16; e += NT) {
            const uint32_t d = S.R[kR - 1 - e], s0 = S.hist[d], c = S.hist[d + 1] - s0;
            for (uint32_t t = s0 + 1; t < s0 + c; ++t) {
                const uint64_t x = B[t];
                uint32_t u = t;
                while (u > s0 && B[u - 1] > x) { B[u] = B[u - 1]; --u; }
                B[u] = x;
            }
        }
        __syncthreads();
        drain(B, scratch, S);
    }
};

}  // namespace lsort_dev
