/*
 * lsort_oracle.c -- CPU ORACLE (test infrastructure only; see lsort_oracle.h).
 *
 * Restates, in plain C, the reference hot path of arXiv 2307.08637 (AIPS2o):
 *   keys.hpp (codec), rng.hpp (splitmix64 Rng), models.hpp/models.cpp
 *   (fit_line, Rmi::train, enforce_monotonic, predict, bucket_index,
 *   SplitterTree, duplicate_fraction), verify.hpp, and the SPEC-only sort
 *   driver.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use it.
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fopenmp).
 */
#include "lsort_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define SIGN_BIT 0x8000000000000000ull

/* ------------------------------------------------------------------ keys */
/* keys.hpp:24-27: non-negative -> flip sign bit, negative -> flip all bits */
uint64_t lso_encode_double(double x) {
    uint64_t b;
    memcpy(&b, &x, 8);
    return (b & SIGN_BIT) ? ~b : (b ^ SIGN_BIT);
}
/* keys.hpp:29-32 */
double lso_decode_double(uint64_t k) {
    uint64_t b = (k & SIGN_BIT) ? (k ^ SIGN_BIT) : ~k;
    double x;
    memcpy(&x, &b, 8);
    return x;
}
/* keys.hpp:36-42: first NaN index or -1 */
int64_t lso_encode_doubles(const double* in, uint64_t* out, size_t n) {
    for (size_t i = 0; i < n; ++i) {
        if (isnan(in[i])) return (int64_t)i;
        out[i] = lso_encode_double(in[i]);
    }
    return -1;
}
/* keys.hpp:44-46 */
void lso_decode_doubles(const uint64_t* in, double* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = lso_decode_double(in[i]);
}

/* ------------------------------------------------------------------- rng */
/* rng.hpp:13-18 */
uint64_t lso_splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
/* rng.hpp:24: next_u64() = splitmix64(state_++) -> draw k of Rng(s) */
uint64_t lso_rng_u64(uint64_t seed, uint64_t draw) { return lso_splitmix64(seed + draw); }
/* rng.hpp:27-29 */
double lso_rng_unit(uint64_t seed, uint64_t draw) {
    return (double)(lso_rng_u64(seed, draw) >> 11) * 0x1.0p-53;
}
/* rng.hpp:32 */
double lso_rng_unit_open(uint64_t seed, uint64_t draw) { return 1.0 - lso_rng_unit(seed, draw); }
/* rng.hpp:35-37 */
uint64_t lso_rng_below(uint64_t seed, uint64_t draw, uint64_t bound) {
    return bound == 0 ? 0 : lso_rng_u64(seed, draw) % bound;
}
/* rng.hpp:41-45: u1 = next_unit_open (draw), u2 = next_unit (draw+1) */
double lso_rng_normal(uint64_t seed, uint64_t draw) {
    double u1 = lso_rng_unit_open(seed, draw);
    double u2 = lso_rng_unit(seed, draw + 1);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}
/* rng.hpp:47-49 */
double lso_rng_exponential(uint64_t seed, uint64_t draw, double lambda) {
    return -log(lso_rng_unit_open(seed, draw)) / lambda;
}

/* ---------------------------------------------------------------- models */
typedef struct { double slope, intercept; } lin_t;

static inline double lin_eval(lin_t m, double x) { return m.slope * x + m.intercept; } /* models.hpp:21 */
static inline double dmax(double a, double b) { return (a < b) ? b : a; }  /* std::max */
static inline double dmin(double a, double b) { return (b < a) ? b : a; }  /* std::min */
static inline double dclamp01(double v) { return (v < 0.0) ? 0.0 : ((1.0 < v) ? 1.0 : v); } /* std::clamp */

/* models.cpp:14-35 fit_line */
static lin_t fit_line(const double* x, const double* y, size_t first, size_t last) {
    size_t n = last - first;
    lin_t r = {0.0, 0.0};
    if (n == 0) return r;
    double sx = 0.0, sy = 0.0;
    for (size_t i = first; i < last; ++i) {
        sx += x[i];
        sy += y[i];
    }
    double mx = sx / (double)n;
    double my = sy / (double)n;
    double sxx = 0.0, sxy = 0.0;
    for (size_t i = first; i < last; ++i) {
        double dx = x[i] - mx;
        sxx += dx * dx;
        sxy += dx * (y[i] - my);
    }
    if (!(sxx > 0.0)) { r.intercept = my; return r; }
    double slope = sxy / sxx;
    if (slope < 0.0) { r.intercept = my; return r; }
    r.slope = slope;
    r.intercept = my - slope * mx;
    return r;
}

#define P_ROOT_S(P) (P)[0]
#define P_ROOT_I(P) (P)[1]
#define P_BASE(P) (P)[2]
#define P_SCALE(P) (P)[3]
#define P_SUB_S(P, m) (P)[4 + 4 * (size_t)(m) + 0]
#define P_SUB_I(P, m) (P)[4 + 4 * (size_t)(m) + 1]
#define P_LO(P, m) (P)[4 + 4 * (size_t)(m) + 2]
#define P_HI(P, m) (P)[4 + 4 * (size_t)(m) + 3]

/* models.hpp:56-58 normalize */
static inline double rmi_normalize(const double* P, uint64_t x) {
    return ((double)x - P_BASE(P)) * P_SCALE(P);
}

/* models.hpp:60-65 route. `i >= B ? B-1 : i` after truncation is written as
 * `t >= B` before it: identical wherever the reference's cast is defined. */
uint32_t lso_rmi_route(const double* P, uint32_t B, double xn) {
    lin_t root = {P_ROOT_S(P), P_ROOT_I(P)};
    double t = lin_eval(root, xn) * (double)B;
    if (!(t > 0.0)) return 0;
    if (t >= (double)B) return B - 1;
    return (uint32_t)t;
}

/* models.hpp:34-43 predict */
double lso_rmi_predict(const double* P, uint32_t B, uint64_t x) {
    double xn = rmi_normalize(P, x);
    uint32_t i = lso_rmi_route(P, B, xn);
    lin_t s = {P_SUB_S(P, i), P_SUB_I(P, i)};
    double v = lin_eval(s, xn);
    if (v < P_LO(P, i)) v = P_LO(P, i);
    if (v > P_HI(P, i)) v = P_HI(P, i);
    if (v < 0.0) v = 0.0;
    if (v > 1.0) v = 1.0;
    return v;
}

/* models.hpp:162-171 PartitionModel::bucket_index (learned branch) with
 * Learned::inv_span (models.hpp:134-137). */
uint32_t lso_learned_bucket(const double* P, uint32_t B, uint32_t bucket_count, double cdf_lo,
                            double cdf_hi, uint64_t x) {
    double f = lso_rmi_predict(P, B, x);
    double s = cdf_hi - cdf_lo;
    double inv_span = s > 0.0 ? 1.0 / s : 0.0;
    double u = (f - cdf_lo) * inv_span;
    double t = u * (double)bucket_count;
    if (!(t > 0.0)) return 0;
    if (t >= (double)bucket_count) return bucket_count - 1;
    return (uint32_t)t;
}

/* models.cpp:75-131 enforce_monotonic */
void lso_enforce_monotonic(double* P, uint32_t B, const uint64_t* s, size_t n) {
    const size_t b = B;
    double* xn = (double*)malloc((n ? n : 1) * sizeof(double));
    for (size_t i = 0; i < n; ++i) xn[i] = rmi_normalize(P, s[i]);

    if (P_ROOT_S(P) < 0.0) {
        lin_t root = {P_ROOT_S(P), P_ROOT_I(P)};
        double mid = n > 0 ? lin_eval(root, xn[n / 2]) : P_ROOT_I(P);
        P_ROOT_S(P) = 0.0;
        P_ROOT_I(P) = mid;
    }
    double* lo = (double*)malloc(b * sizeof(double));
    double* hi = (double*)malloc(b * sizeof(double));
    unsigned char* nonempty = (unsigned char*)calloc(b, 1);
    for (size_t m = 0; m < b; ++m) { lo[m] = -INFINITY; hi[m] = INFINITY; }
    size_t begin = 0;
    for (size_t m = 0; m < b && begin < n; ++m) {
        size_t end = begin;
        while (end < n && lso_rmi_route(P, B, xn[end]) == m) ++end;
        if (end > begin) {
            nonempty[m] = 1;
            if (P_SUB_S(P, m) < 0.0) {
                lin_t sm = {P_SUB_S(P, m), P_SUB_I(P, m)};
                double v = lin_eval(sm, xn[begin + (end - begin) / 2]);
                P_SUB_S(P, m) = 0.0;
                P_SUB_I(P, m) = v;
            }
            lin_t sm = {P_SUB_S(P, m), P_SUB_I(P, m)};
            lo[m] = lin_eval(sm, xn[begin]);
            hi[m] = lin_eval(sm, xn[end - 1]);
        }
        begin = end;
    }
    for (size_t m = 1; m < b; ++m) lo[m] = dmax(lo[m], lo[m - 1]);
    for (size_t m = b - 1; m-- > 0;) hi[m] = dmin(hi[m], hi[m + 1]);
    for (size_t m = 0; m + 1 < b; ++m) hi[m] = dmin(hi[m], lo[m + 1]);
    for (size_t m = 0; m < b; ++m) hi[m] = dmax(hi[m], lo[m]);
    for (size_t m = 0; m < b; ++m) {
        lo[m] = dclamp01(lo[m]);
        hi[m] = dclamp01(hi[m]);
    }
    lo[0] = 0.0;
    hi[b - 1] = 1.0;
    for (size_t m = 0; m < b; ++m) {
        if (!nonempty[m]) {
            P_SUB_S(P, m) = 0.0;
            P_SUB_I(P, m) = 0.5 * (lo[m] + hi[m]);
        }
        P_LO(P, m) = lo[m];
        P_HI(P, m) = hi[m];
    }
    free(xn);
    free(lo);
    free(hi);
    free(nonempty);
}

/* Rmi::train from the slice loop on (models.cpp:58-72), for a given root
 * model: the test hook that checks a GPU-trained RMI whose root came from a
 * parallel (not sequential) sum against the reference's own slicing and
 * per-slice fits. P[0..1] (root) must be set by the caller. */
int lso_rmi_train_given_root(const uint64_t* s, size_t n, uint32_t B, double* P) {
    if (n < 2 || B == 0) return -1;
    P_BASE(P) = (double)s[0];
    double key_max = (double)s[n - 1];
    P_SCALE(P) = key_max > P_BASE(P) ? 1.0 / (key_max - P_BASE(P)) : 0.0;
    double* xn = (double*)malloc(n * sizeof(double));
    double* tg = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) {
        xn[i] = rmi_normalize(P, s[i]);
        tg[i] = (double)i / (double)n;
    }
    for (uint32_t m = 0; m < B; ++m) {
        P_SUB_S(P, m) = 0.0;
        P_SUB_I(P, m) = 0.0;
        P_LO(P, m) = 0.0;
        P_HI(P, m) = 1.0;
    }
    size_t begin = 0;
    for (size_t m = 0; m < B && begin < n; ++m) {
        size_t end = begin;
        while (end < n && lso_rmi_route(P, B, xn[end]) == m) ++end;
        if (end > begin) {
            lin_t f = fit_line(xn, tg, begin, end);
            P_SUB_S(P, m) = f.slope;
            P_SUB_I(P, m) = f.intercept;
        }
        begin = end;
    }
    free(xn);
    free(tg);
    lso_enforce_monotonic(P, B, s, n);
    return 0;
}

/* models.cpp:39-73 Rmi::train. Returns -1 on the reference's
 * std::invalid_argument preconditions (n < 2, B == 0). */
int lso_rmi_train(const uint64_t* s, size_t n, uint32_t B, double* P) {
    if (n < 2 || B == 0) return -1;
    P_BASE(P) = (double)s[0];
    double key_max = (double)s[n - 1];
    P_SCALE(P) = key_max > P_BASE(P) ? 1.0 / (key_max - P_BASE(P)) : 0.0;
    double* xn = (double*)malloc(n * sizeof(double));
    double* tg = (double*)malloc(n * sizeof(double));
    for (size_t i = 0; i < n; ++i) {
        xn[i] = rmi_normalize(P, s[i]);
        tg[i] = (double)i / (double)n;
    }
    lin_t root = fit_line(xn, tg, 0, n);
    P_ROOT_S(P) = root.slope;
    P_ROOT_I(P) = root.intercept;
    for (uint32_t m = 0; m < B; ++m) {
        P_SUB_S(P, m) = 0.0;
        P_SUB_I(P, m) = 0.0;
        P_LO(P, m) = 0.0;
        P_HI(P, m) = 1.0;
    }
    size_t begin = 0;
    for (size_t m = 0; m < B && begin < n; ++m) {
        size_t end = begin;
        while (end < n && lso_rmi_route(P, B, xn[end]) == m) ++end;
        if (end > begin) {
            lin_t f = fit_line(xn, tg, begin, end);
            P_SUB_S(P, m) = f.slope;
            P_SUB_I(P, m) = f.intercept;
        }
        begin = end;
    }
    free(xn);
    free(tg);
    lso_enforce_monotonic(P, B, s, n);
    return 0;
}

/* ---------------------------------------------------------- SplitterTree */
static size_t count_equal(const uint64_t* s, size_t n, uint64_t v) { /* std::equal_range */
    size_t lo = 0, hi = n;
    while (lo < hi) { size_t mid = lo + (hi - lo) / 2; if (s[mid] < v) lo = mid + 1; else hi = mid; }
    size_t first = lo;
    hi = n;
    while (lo < hi) { size_t mid = lo + (hi - lo) / 2; if (v < s[mid]) hi = mid; else lo = mid + 1; }
    return lo - first;
}

static void tree_fill(lso_tree* t, const uint64_t* padded, size_t node, size_t* next) {
    if (node >= t->leaf_origin) return;
    tree_fill(t, padded, 2 * node, next);
    t->tree[node] = padded[(*next)++];
    tree_fill(t, padded, 2 * node + 1, next);
}

/* models.cpp:133-185 SplitterTree::build */
int lso_tree_build(const uint64_t* s, size_t n, uint32_t budget, int equality_mode, lso_tree* t) {
    if (n == 0) return -1;
    if (budget < 2 || (budget & (budget - 1)) != 0 || budget > LSO_MAX_TREE) return -1;
    const size_t k = budget;
    memset(t, 0, sizeof(*t));
    size_t m = 0;
    for (size_t i = 0; i + 1 < k; ++i) {
        size_t q = (i + 1) * n / k;
        size_t pos = (q > 1 ? q : 1) - 1;
        uint64_t v = s[pos];
        if (m == 0 || v > t->splitters[m - 1]) t->splitters[m++] = v;
    }
    if (m == 0) t->splitters[m++] = s[0];
    t->nsplitters = (uint32_t)m;
    t->eq_offset[0] = 0;
    for (size_t i = 0; i < m; ++i) {
        size_t count = count_equal(s, n, t->splitters[i]);
        int heavy = equality_mode && count * k > n;
        t->eq_offset[i + 1] = t->eq_offset[i] + (heavy ? 2u : 1u);
    }
    t->bucket_count = t->eq_offset[m] + 1;
    uint32_t levels = 1;
    while (((size_t)1 << levels) < m + 1) ++levels;
    t->levels = levels;
    t->leaf_origin = 1u << levels;
    uint64_t padded[LSO_MAX_TREE];
    for (size_t i = 0; i + 1 < t->leaf_origin; ++i) padded[i] = i < m ? t->splitters[i] : UINT64_MAX;
    t->tree[0] = 0;
    size_t next = 0;
    tree_fill(t, padded, 1, &next);
    return 0;
}

/* models.hpp:92-101 SplitterTree::classify */
uint32_t lso_tree_classify(const lso_tree* t, uint64_t x) {
    uint32_t i = 1;
    for (uint32_t lvl = 0; lvl < t->levels; ++lvl) i = 2 * i + (x > t->tree[i] ? 1u : 0u);
    uint32_t base = i - t->leaf_origin;
    uint32_t eq = (base < t->nsplitters) && (t->eq_offset[base + 1] - t->eq_offset[base] > 1) &&
                  (x == t->splitters[base]);
    return t->eq_offset[base] + eq;
}

/* Bulk forms of the two classifiers above (one call per array; test helpers). */
void lso_learned_bucket_many(const double* P, uint32_t B, uint32_t bucket_count, double cdf_lo, double cdf_hi,
                             const uint64_t* x, size_t n, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = lso_learned_bucket(P, B, bucket_count, cdf_lo, cdf_hi, x[i]);
}
void lso_tree_classify_many(const lso_tree* t, const uint64_t* x, size_t n, uint32_t* out) {
    for (size_t i = 0; i < n; ++i) out[i] = lso_tree_classify(t, x[i]);
}

/* models.cpp:187-193 */
double lso_duplicate_fraction(const uint64_t* s, size_t n) {
    if (n == 0) return 0.0;
    size_t distinct = 1;
    for (size_t i = 1; i < n; ++i) distinct += s[i] != s[i - 1];
    return 1.0 - (double)distinct / (double)n;
}

/* ---------------------------------------------------------------- verify */
int lso_verify_sorted(const uint64_t* a, size_t n, uint64_t* fv) { /* verify.hpp:17-22 */
    for (size_t i = 1; i < n; ++i)
        if (a[i - 1] > a[i]) { if (fv) *fv = i; return 0; }
    if (fv) *fv = 0;
    return 1;
}
uint64_t lso_multiset_hash(const uint64_t* a, size_t n) { /* verify.hpp:25-29 */
    uint64_t h = 0;
    for (size_t i = 0; i < n; ++i) h += lso_splitmix64(a[i]);
    return h;
}

/* ------------------------------------------------------------ generators */
int lso_gen_is_float(int d) {
    return d == LSO_GEN_UNIFORM || d == LSO_GEN_NORMAL || d == LSO_GEN_LOGNORMAL05 ||
           d == LSO_GEN_EXPONENTIAL2 || d == LSO_GEN_MIXGAUSS || d == LSO_GEN_LOGNORMAL2;
}

static uint64_t isqrt_u64(uint64_t n) {
    uint64_t r = (uint64_t)sqrt((double)n);
    while (r * r > n) --r;
    while ((r + 1) * (r + 1) <= n) ++r;
    return r;
}

/* Fisher-Yates with Rng(seed) starting at draw `d0`: for i = n-1..1,
 * j = next_below(i+1), swap(a[i], a[j]). */
static void fisher_yates(uint64_t* a, uint64_t n, uint64_t seed, uint64_t d0) {
    uint64_t d = d0;
    for (uint64_t i = n; i-- > 1;) {
        uint64_t j = lso_rng_below(seed, d++, i + 1);
        uint64_t tmp = a[i];
        a[i] = a[j];
        a[j] = tmp;
    }
}

#define ZIPF_M 1000000u

int lso_generate(int dist, uint64_t total, uint64_t seed, uint64_t first, uint64_t count, void* out,
                 int threads) {
    if (first + count > total) return -1;
    int shuffled = dist == LSO_GEN_ROOTDUPS || dist == LSO_GEN_TWODUPS || dist == LSO_GEN_ZIPF;
    if (shuffled && (first != 0 || count != total)) return -1;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#else
    (void)threads;
#endif
    double* od = (double*)out;
    uint64_t* ou = (uint64_t*)out;
    int64_t cnt = (int64_t)count;
    switch (dist) {
    case LSO_GEN_UNIFORM:
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) od[k] = lso_rng_unit(seed, first + k);
        return 0;
    case LSO_GEN_NORMAL:
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) od[k] = lso_rng_normal(seed, 2 * (first + k));
        return 0;
    case LSO_GEN_LOGNORMAL05:
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) od[k] = exp(0.5 * lso_rng_normal(seed, 2 * (first + k)));
        return 0;
    case LSO_GEN_EXPONENTIAL2:
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) od[k] = lso_rng_exponential(seed, first + k, 2.0);
        return 0;
    case LSO_GEN_LOGNORMAL2:
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) od[k] = exp(2.0 * lso_rng_normal(seed, 2 * (first + k)));
        return 0;
    case LSO_GEN_MIXGAUSS: {
        double mu[5], sd[5];
        for (int c = 0; c < 5; ++c) {
            mu[c] = -100.0 + 200.0 * lso_rng_unit(seed, 2 * c);
            sd[c] = 1.0 + 4.0 * lso_rng_unit(seed, 2 * c + 1);
        }
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) {
            uint64_t d = 10 + 3 * (first + k);
            uint64_t c = lso_rng_below(seed, d, 5);
            od[k] = mu[c] + sd[c] * lso_rng_normal(seed, d + 1);
        }
        return 0;
    }
    case LSO_GEN_ROOTDUPS: {
        uint64_t r = isqrt_u64(total);
        if (r == 0) r = 1;
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) ou[k] = (uint64_t)k % r;
        fisher_yates(ou, total, seed, 0);
        return 0;
    }
    case LSO_GEN_TWODUPS: {
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) {
            unsigned __int128 v = (unsigned __int128)(uint64_t)k * (uint64_t)k + total / 2;
            ou[k] = (uint64_t)(v % total);
        }
        fisher_yates(ou, total, seed, 0);
        return 0;
    }
    case LSO_GEN_ZIPF: {
        double* cdf = (double*)malloc(ZIPF_M * sizeof(double));
        double h = 0.0;
        for (uint32_t r = 1; r <= ZIPF_M; ++r) h += 1.0 / pow((double)r, 0.75);
        double acc = 0.0;
        for (uint32_t r = 1; r <= ZIPF_M; ++r) {
            acc += 1.0 / pow((double)r, 0.75);
            cdf[r - 1] = acc / h;
        }
#pragma omp parallel for num_threads(threads) schedule(static)
        for (int64_t k = 0; k < cnt; ++k) {
            double u = lso_rng_unit(seed, (uint64_t)k);
            size_t lo = 0, hi = ZIPF_M; /* upper_bound */
            while (lo < hi) { size_t mid = (lo + hi) / 2; if (u < cdf[mid]) hi = mid; else lo = mid + 1; }
            uint64_t key = (uint64_t)lo + 1;
            ou[k] = key > ZIPF_M ? ZIPF_M : key;
        }
        free(cdf);
        fisher_yates(ou, total, seed, total);
        return 0;
    }
    default:
        return -1;
    }
}

/* ----------------------------------------------------------- sort driver */
void lso_cfg_default(lso_cfg* c) {
    c->rmi_bucket_count = 1024;
    c->tree_bucket_count = 256;
    c->min_rmi_input = 100000;
    c->max_duplicate_fraction = 0.10;
    c->radix_base_case = 4096;
    c->insertion_base_case = 16;
    c->first_sample_cap = 2 * 256 * 16;
    c->rmi_sample_cap = 1u << 20;
    c->sample_fraction = 0.01;
    c->seed = 0x5EEDull;
    c->workers = 0;
}

/* Sampling stream of a segment (no reference code; SPEC.md:438 sizes). */
uint64_t lso_seg_seed(uint64_t cfg_seed, uint64_t seg_begin, uint32_t depth) {
    return lso_splitmix64(cfg_seed ^ lso_splitmix64(seg_begin + ((uint64_t)depth << 48)));
}
/* ceil(min(0.01 N, 2*tree_bucket_count*16)), at least 2 */
uint64_t lso_first_sample_size(const lso_cfg* c, uint64_t n) {
    double v = c->sample_fraction * (double)n;
    double cap = (double)c->first_sample_cap;
    uint64_t s = (uint64_t)ceil(v < cap ? v : cap);
    return s < 2 ? 2 : s;
}
/* min(0.01 N, 2^20) (ceil), at least 2 */
uint64_t lso_rmi_sample_size(const lso_cfg* c, uint64_t n) {
    double v = c->sample_fraction * (double)n;
    double cap = (double)c->rmi_sample_cap;
    uint64_t s = (uint64_t)ceil(v < cap ? v : cap);
    return s < 2 ? 2 : s;
}

static void insertion_sort(uint64_t* a, uint64_t n) {
    for (uint64_t i = 1; i < n; ++i) {
        uint64_t v = a[i];
        uint64_t j = i;
        while (j > 0 && a[j - 1] > v) { a[j] = a[j - 1]; --j; }
        a[j] = v;
    }
}

/* MSD byte radix from byte `shift` down. */
static void msd_radix(uint64_t* a, uint64_t* tmp, uint64_t n, int shift, uint32_t ins) {
    if (n <= ins) { insertion_sort(a, n); return; }
    if (shift < 0) return;
    uint64_t cnt[257];
    memset(cnt, 0, sizeof(cnt));
    for (uint64_t i = 0; i < n; ++i) cnt[((a[i] >> shift) & 0xFF) + 1]++;
    if (cnt[((a[0] >> shift) & 0xFF) + 1] == n) { msd_radix(a, tmp, n, shift - 8, ins); return; }
    for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
    uint64_t pos[256];
    memcpy(pos, cnt, sizeof(pos));
    for (uint64_t i = 0; i < n; ++i) tmp[pos[(a[i] >> shift) & 0xFF]++] = a[i];
    memcpy(a, tmp, n * sizeof(uint64_t));
    for (int b = 0; b < 256; ++b) {
        uint64_t len = cnt[b + 1] - cnt[b];
        if (len > 1) msd_radix(a + cnt[b], tmp, len, shift - 8, ins);
    }
}

void lso_radix_base_case_sort(uint64_t* a, uint64_t n, uint32_t ins) {
    if (n < 2) return;
    uint64_t stackbuf[4096];
    uint64_t* tmp = n <= 4096 ? stackbuf : (uint64_t*)malloc(n * sizeof(uint64_t));
    msd_radix(a, tmp, n, 56, ins);
    if (tmp != stackbuf) free(tmp);
}

/* heapsort: the depth-cap comparison fallback */
static void sift_down(uint64_t* a, uint64_t start, uint64_t n) {
    uint64_t r = start;
    for (;;) {
        uint64_t c = 2 * r + 1;
        if (c >= n) return;
        if (c + 1 < n && a[c] < a[c + 1]) ++c;
        if (a[r] >= a[c]) return;
        uint64_t t = a[r]; a[r] = a[c]; a[c] = t;
        r = c;
    }
}
static void heap_sort(uint64_t* a, uint64_t n) {
    if (n < 2) return;
    for (uint64_t s = n / 2; s-- > 0;) sift_down(a, s, n);
    for (uint64_t e = n - 1; e > 0; --e) {
        uint64_t t = a[0]; a[0] = a[e]; a[e] = t;
        sift_down(a, 0, e);
    }
}

int lso_build_partition_model(const uint64_t* a, uint64_t n, uint64_t seg_begin, uint32_t depth,
                              const lso_cfg* c, uint32_t rmi_buckets, uint32_t tree_buckets,
                              int* kind_out, double* P, lso_tree* tree, double* dup_out) {
    uint64_t seed = lso_seg_seed(c->seed, seg_begin, depth);
    uint64_t s1 = lso_first_sample_size(c, n);
    uint64_t* smp = (uint64_t*)malloc(s1 * sizeof(uint64_t));
    for (uint64_t j = 0; j < s1; ++j) smp[j] = a[lso_rng_below(seed, j, n)];
    lso_radix_base_case_sort(smp, s1, 16);
    double dup = lso_duplicate_fraction(smp, s1);
    if (dup_out) *dup_out = dup;
    if (n >= c->min_rmi_input && dup <= c->max_duplicate_fraction) {
        uint64_t s2 = lso_rmi_sample_size(c, n);
        uint64_t* smp2 = (uint64_t*)malloc(s2 * sizeof(uint64_t));
        for (uint64_t j = 0; j < s2; ++j) smp2[j] = a[lso_rng_below(seed, s1 + j, n)];
        lso_radix_base_case_sort(smp2, s2, 16);
        lso_rmi_train(smp2, s2, rmi_buckets, P);
        free(smp2);
        *kind_out = 0;
    } else {
        lso_tree_build(smp, s1, tree_buckets, 1, tree);
        *kind_out = 1;
    }
    free(smp);
    return 0;
}

typedef struct {
    const lso_cfg* c;
    uint32_t depth_cap;
} sort_ctx;

static int all_equal(const uint64_t* a, uint64_t n) {
    for (uint64_t i = 1; i < n; ++i)
        if (a[i] != a[0]) return 0;
    return 1;
}

/* Data in x[0,n); the sorted result must end in x (want_x) or y. */
static void sort_rec(const sort_ctx* sc, uint64_t* x, uint64_t* y, uint64_t n, uint64_t seg_begin,
                     uint32_t depth, int want_x) {
    const lso_cfg* c = sc->c;
    if (n <= c->radix_base_case || n < 2) {
        lso_radix_base_case_sort(x, n, c->insertion_base_case);
        if (!want_x) memcpy(y, x, n * sizeof(uint64_t));
        return;
    }
    if (depth > sc->depth_cap) {
        heap_sort(x, n);
        if (!want_x) memcpy(y, x, n * sizeof(uint64_t));
        return;
    }
    int kind;
    uint32_t B = c->rmi_bucket_count;
    double* P = (double*)malloc((4 + 4 * (size_t)B) * sizeof(double));
    lso_tree* tree = (lso_tree*)malloc(sizeof(lso_tree));
    lso_build_partition_model(x, n, seg_begin, depth, c, B, c->tree_bucket_count, &kind, P, tree, NULL);
    uint32_t nb = kind == 0 ? B : tree->bucket_count;

    /* classify_and_flush, restated out of place: chunked
     * classification with per-chunk histograms, then a stable scatter. */
    uint16_t* id = (uint16_t*)malloc(n * sizeof(uint16_t));
    int par = n >= (1u << 20);
    int64_t nchunk = 1;
#ifdef _OPENMP
    if (par) nchunk = (int64_t)omp_get_num_threads() * 4;
#endif
    uint64_t* hist = (uint64_t*)calloc((size_t)nchunk * nb, sizeof(uint64_t));
#pragma omp taskloop if (par) grainsize(1)
    for (int64_t ch = 0; ch < nchunk; ++ch) {
        uint64_t* h = hist + (size_t)ch * nb;
        uint64_t lo = n * (uint64_t)ch / (uint64_t)nchunk, hi = n * (uint64_t)(ch + 1) / (uint64_t)nchunk;
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t b = kind == 0 ? lso_learned_bucket(P, B, B, 0.0, 1.0, x[i])
                                   : lso_tree_classify(tree, x[i]);
            id[i] = (uint16_t)b;
            h[b]++;
        }
    }
    uint64_t* start = (uint64_t*)malloc((nb + 1) * sizeof(uint64_t));
    uint64_t acc = 0;
    for (uint32_t b = 0; b < nb; ++b) {
        start[b] = acc;
        for (int64_t ch = 0; ch < nchunk; ++ch) {
            uint64_t v = hist[(size_t)ch * nb + b];
            hist[(size_t)ch * nb + b] = acc;
            acc += v;
        }
    }
    start[nb] = acc;
#pragma omp taskloop if (par) grainsize(1)
    for (int64_t ch = 0; ch < nchunk; ++ch) {
        uint64_t* h = hist + (size_t)ch * nb;
        uint64_t lo = n * (uint64_t)ch / (uint64_t)nchunk, hi = n * (uint64_t)(ch + 1) / (uint64_t)nchunk;
        for (uint64_t i = lo; i < hi; ++i) y[h[id[i]]++] = x[i];
    }
    free(id);
    free(hist);

    /* mark_homogeneous + recursion */
    for (uint32_t b = 0; b < nb; ++b) {
        uint64_t len = start[b + 1] - start[b];
        if (len == 0) continue;
        uint64_t* cy = y + start[b];
        uint64_t* cx = x + start[b];
        int homogeneous = 0;
        if (kind == 1) {
            /* equality bucket of a heavy splitter: all keys equal */
            for (uint32_t s = 0; s < tree->nsplitters; ++s)
                if (tree->eq_offset[s + 1] - tree->eq_offset[s] > 1 && tree->eq_offset[s] + 1 == b)
                    homogeneous = 1;
        }
        if (!homogeneous && cy[0] == cy[len - 1] && all_equal(cy, len)) homogeneous = 1;
        if (homogeneous) {
            if (want_x) memcpy(cx, cy, len * sizeof(uint64_t));
            continue;
        }
        /* child data in y; result must end in x iff want_x */
        uint32_t cdepth = depth + 1;
        if (len == n) cdepth = sc->depth_cap + 1; /* no progress: force the fallback */
        if (len > 2u * c->radix_base_case) {
#pragma omp task firstprivate(cy, cx, len, b, cdepth)
            sort_rec(sc, cy, cx, len, seg_begin + start[b], cdepth, !want_x);
        } else {
            sort_rec(sc, cy, cx, len, seg_begin + start[b], cdepth, !want_x);
        }
    }
#pragma omp taskwait
    free(start);
    free(P);
    free(tree);
}

int lso_sort_keys(uint64_t* a, uint64_t n, const lso_cfg* c) {
    if (n < 2) return 0;
    sort_ctx sc;
    sc.c = c;
    sc.depth_cap = (uint32_t)ceil(log2((double)n) / log2((double)c->tree_bucket_count)) + 4;
    uint64_t* tmp = (uint64_t*)malloc(n * sizeof(uint64_t));
#ifdef _OPENMP
    int nth = c->workers ? (int)c->workers : omp_get_max_threads();
#pragma omp parallel num_threads(nth)
#pragma omp single
#endif
    sort_rec(&sc, a, tmp, n, 0, 0, 1);
    free(tmp);
    return 0;
}

int lso_sort_doubles(double* a, uint64_t n, const lso_cfg* c, int64_t* nan_index) {
    uint64_t* k = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    int64_t bad = lso_encode_doubles(a, k, n);
    if (nan_index) *nan_index = bad;
    if (bad >= 0) { free(k); return 2; }
    lso_sort_keys(k, n, c);
    lso_decode_doubles(k, a, n);
    free(k);
    return 0;
}

/* --------------------------------------- LearnedSort 2.0 classic path */
/* model_counting_sort: predicted position of x in a segment
 * of len keys = PartitionModel::bucket_index with bucket_count = len over the
 * segment's CDF range [cdf_lo, cdf_hi) (models.hpp:128-138,162-171), i.e.
 * floor(len * F(x)) within the range; stable counting placement (ties keep
 * the input order). Sorted iff the model is monotone and collision-free. */
void lso_model_counting_sort(const uint64_t* a, size_t n, const double* P, uint32_t B, double cdf_lo,
                             double cdf_hi, uint64_t* out) {
    if (n == 0) return;
    uint32_t* pos = (uint32_t*)malloc(n * sizeof(uint32_t));
    size_t* start = (size_t*)calloc(n + 1, sizeof(size_t));
    for (size_t i = 0; i < n; ++i) {
        pos[i] = lso_learned_bucket(P, B, (uint32_t)n, cdf_lo, cdf_hi, a[i]);
        start[pos[i] + 1]++;
    }
    for (size_t p = 0; p < n; ++p) start[p + 1] += start[p];
    for (size_t i = 0; i < n; ++i) out[start[pos[i]]++] = a[i];
    free(pos);
    free(start);
}

/* learned_sort_classic (§2.2, §3.3): one RMI on a
 * 1% sample (Rng(seed).next_below, capped at rmi_sample_cap); round 1 into B
 * buckets; round 2 of every bucket b into B sub-buckets with the SAME model
 * restricted to the CDF range [b/B, (b+1)/B); model_counting_sort of every
 * sub-bucket over its CDF range [b/B + j/B^2, b/B + (j+1)/B^2); one final
 * insertion-sort sweep. stats (nullable): [0] non-empty sub-buckets after
 * round two, [1] swaps made by the final insertion sort. */
int lso_learned_sort_classic(uint64_t* a, uint64_t n, const lso_cfg* c, uint64_t* stats) {
    if (stats) { stats[0] = 0; stats[1] = 0; }
    if (n < 2) return 0;
    const uint32_t B = c->rmi_bucket_count;
    const uint64_t s = lso_rmi_sample_size(c, n);
    uint64_t* smp = (uint64_t*)malloc(s * sizeof(uint64_t));
    for (uint64_t j = 0; j < s; ++j) smp[j] = a[lso_rng_below(c->seed, j, n)];
    lso_radix_base_case_sort(smp, s, 16);
    double* P = (double*)malloc((4 + 4 * (size_t)B) * sizeof(double));
    lso_rmi_train(smp, s, B, P);
    free(smp);
    const uint64_t BB = (uint64_t)B * B;
    uint32_t* q = (uint32_t*)malloc(n * sizeof(uint32_t));  /* b * B + j */
    uint64_t* cnt = (uint64_t*)calloc(BB + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t b = lso_learned_bucket(P, B, B, 0.0, 1.0, a[i]);
        const uint32_t j = lso_learned_bucket(P, B, B, (double)b / B, (double)(b + 1) / B, a[i]);
        q[i] = b * B + j;
        cnt[q[i] + 1]++;
    }
    for (uint64_t k = 0; k < BB; ++k) {
        if (stats && cnt[k + 1]) stats[0]++;
        cnt[k + 1] += cnt[k];
    }
    uint64_t* y = (uint64_t*)malloc(n * sizeof(uint64_t));
    uint64_t* cur = (uint64_t*)malloc((BB + 1) * sizeof(uint64_t));
    memcpy(cur, cnt, (BB + 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) y[cur[q[i]]++] = a[i];
    free(cur);
    free(q);
    for (uint64_t k = 0; k < BB; ++k) {
        const uint64_t lo = cnt[k], len = cnt[k + 1] - lo;
        if (len == 0) continue;
        const uint32_t b = (uint32_t)(k / B), j = (uint32_t)(k % B);
        const double c0 = (double)b / B + (double)j / (double)BB;
        lso_model_counting_sort(y + lo, len, P, B, c0, c0 + 1.0 / (double)BB, a + lo);
    }
    free(cnt);
    free(y);
    free(P);
    /* insertion-sort sweep (§2.2: corrects the RMI's mistakes) */
    uint64_t swaps = 0;
    for (uint64_t i = 1; i < n; ++i) {
        const uint64_t x = a[i];
        uint64_t u = i;
        while (u > 0 && a[u - 1] > x) { a[u] = a[u - 1]; --u; ++swaps; }
        a[u] = x;
    }
    if (stats) stats[1] = swaps;
    return 0;
}

/* ------------------------------------------------ pivot analysis */
/* PAPER.md:324-349 (Alg. 4) */
size_t lso_learned_pivots(const uint64_t* a, size_t n, const double* P, uint32_t B, uint32_t b, uint64_t* out) {
    if (b < 2) return 0;
    uint64_t* mx = (uint64_t*)calloc(b, sizeof(uint64_t));
    unsigned char* hit = (unsigned char*)calloc(b, 1);
    for (size_t w = 0; w < n; ++w) {
        const uint32_t g = lso_learned_bucket(P, B, b, 0.0, 1.0, a[w]);
        if (!hit[g] || a[w] > mx[g]) { mx[g] = a[w]; hit[g] = 1; }
    }
    size_t np = 0;
    for (uint32_t i = 0; i + 1 < b; ++i)
        if (hit[i] && (np == 0 || mx[i] > out[np - 1])) out[np++] = mx[i];
    free(mx);
    free(hit);
    return np;
}

uint64_t lso_rank_le(const uint64_t* s, size_t n, uint64_t p) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = lo + (hi - lo) / 2;
        if (s[mid] <= p) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* sum_{i=0}^{B-2} |P(A <= p_i) - (i+1)/B| */
double lso_pivot_quality(const uint64_t* s, size_t n, const uint64_t* pv, size_t np, uint32_t b) {
    if (np + 1 != b || n == 0) return -1.0;
    double d = 0.0;
    for (size_t i = 0; i < np; ++i) {
        const double c = (double)lso_rank_le(s, n, pv[i]) / (double)n;
        const double t = (double)(i + 1) / (double)b;
        d += c > t ? c - t : t - c;
    }
    return d;
}

/* PAPER.md §3.1: eta = max(P(A <= p), 1 - P(A <= p)) - 1/2 */
double lso_eta(const uint64_t* s, size_t n, uint64_t p) {
    if (n == 0) return 0.0;
    const double c = (double)lso_rank_le(s, n, p) / (double)n;
    const double o = 1.0 - c;
    return (c > o ? c : o) - 0.5;
}
