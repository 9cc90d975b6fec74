// gen.cpp -- host-side synthetic key generators for the BASELINE.json configs
// (data.generate; dataset definitions).
//
// Every draw comes from the reference's counter-based PRNG: draw k of
// Rng(seed) is splitmix64(seed + k) (rng.hpp:13-49), so elements are
// generated independently and in parallel (OpenMP) with glibc libm, bit-
// identical to a sequential Rng walk. Inputs are generated on the host
// because CUDA's log/cos are not bit-identical to glibc (hard
// part 6).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/lsort_cuda.h"

namespace {

inline uint64_t sm64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
struct Draw {  // Rng(seed) at stream position k
    uint64_t seed;
    uint64_t u64(uint64_t k) const { return sm64(seed + k); }
    double unit(uint64_t k) const { return static_cast<double>(u64(k) >> 11) * 0x1.0p-53; }
    double unit_open(uint64_t k) const { return 1.0 - unit(k); }
    uint64_t below(uint64_t k, uint64_t bound) const { return bound == 0 ? 0 : u64(k) % bound; }
    double normal(uint64_t k) const {  // rng.hpp:41-45, draws k and k+1
        double u1 = unit_open(k);
        double u2 = unit(k + 1);
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
    }
    double exponential(uint64_t k, double lambda) const { return -std::log(unit_open(k)) / lambda; }
};

uint64_t isqrt(uint64_t n) {
    uint64_t r = (uint64_t)std::sqrt((double)n);
    while (r * r > n) --r;
    while ((r + 1) * (r + 1) <= n) ++r;
    return r;
}

void shuffle(uint64_t* a, uint64_t n, const Draw& d, uint64_t k0) {  // Fisher-Yates, i = n-1..1
    uint64_t k = k0;
    for (uint64_t i = n; i-- > 1;) {
        uint64_t j = d.below(k++, i + 1);
        uint64_t t = a[i];
        a[i] = a[j];
        a[j] = t;
    }
}

}  // namespace

extern "C" int lsort_gen_keys(int dist, uint64_t total, uint64_t seed, uint64_t first, uint64_t count, void* out,
                              int threads) {
    if (first + count > total || (count && !out)) return LSORT_EINVAL;
    const bool shuffled = dist == 5 || dist == 6 || dist == 7;
    if (shuffled && (first != 0 || count != total)) return LSORT_EINVAL;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    (void)threads;
#endif
    const Draw D{seed};
    double* od = static_cast<double*>(out);
    uint64_t* ou = static_cast<uint64_t*>(out);
    const int64_t cnt = (int64_t)count;
    switch (dist) {
    case 0:  // Uniform[0,1)
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) od[i] = D.unit(first + i);
        return LSORT_OK;
    case 1:  // Normal(0,1)
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) od[i] = D.normal(2 * (first + i));
        return LSORT_OK;
    case 2:  // LogNormal(0, 0.5)
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) od[i] = std::exp(0.5 * D.normal(2 * (first + i)));
        return LSORT_OK;
    case 3:  // Exponential(2)
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) od[i] = D.exponential(first + i, 2.0);
        return LSORT_OK;
    case 8:  // LogNormal(0, 2)
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) od[i] = std::exp(2.0 * D.normal(2 * (first + i)));
        return LSORT_OK;
    case 4: {  // equal-weight mixture of 5 Gaussians (BASELINE.json config 3)
        double mu[5], sd[5];
        for (int c = 0; c < 5; ++c) {
            mu[c] = -100.0 + 200.0 * D.unit(2 * c);
            sd[c] = 1.0 + 4.0 * D.unit(2 * c + 1);
        }
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) {
            const uint64_t k = 10 + 3 * (first + i);
            const uint64_t c = D.below(k, 5);
            od[i] = mu[c] + sd[c] * D.normal(k + 1);
        }
        return LSORT_OK;
    }
    case 5: {  // root dups: A[i] = i mod floor(sqrt(N)), shuffled
        uint64_t r = isqrt(total);
        if (r == 0) r = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) ou[i] = (uint64_t)i % r;
        shuffle(ou, total, D, 0);
        return LSORT_OK;
    }
    case 6: {  // two dups: A[i] = (i*i + N/2) mod N, shuffled
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) {
            unsigned __int128 v = (unsigned __int128)(uint64_t)i * (uint64_t)i + total / 2;
            ou[i] = (uint64_t)(v % total);
        }
        shuffle(ou, total, D, 0);
        return LSORT_OK;
    }
    case 7: {  // Zipf(s = 0.75) over 1e6 ranks, inverse CDF, shuffled
        const uint32_t M = 1000000;
        std::vector<double> cdf(M);
        double h = 0.0;
        for (uint32_t r = 1; r <= M; ++r) h += 1.0 / std::pow((double)r, 0.75);
        double acc = 0.0;
        for (uint32_t r = 1; r <= M; ++r) {
            acc += 1.0 / std::pow((double)r, 0.75);
            cdf[r - 1] = acc / h;
        }
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t i = 0; i < cnt; ++i) {
            const double u = D.unit((uint64_t)i);
            size_t lo = 0, hi = M;  // upper_bound
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (u < cdf[mid]) hi = mid; else lo = mid + 1;
            }
            uint64_t key = (uint64_t)lo + 1;
            ou[i] = key > M ? M : key;
        }
        shuffle(ou, total, D, total);
        return LSORT_OK;
    }
    default:
        return LSORT_EINVAL;
    }
}
