/*
 * lsort_oracle.h -- CPU ORACLE (test infrastructure only).
 *
 * Plain-C restatement of the reference's sort hot path (arXiv 2307.08637,
 * parallel LearnedSort / AIPS2o) used as the CHECKER for the CUDA library.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it. The product path (paper_2307_08637_b200)
 * never links or calls anything in oracle/.
 *
 * Each function cites the reference file:line it restates
 * (paths relative to /root/reference/proj/src/ unless noted).
 * Compiled with -O2 -ffp-contract=off so the double arithmetic matches the
 * reference's Release build bit for bit.
 *
 * Parity pinning: the model layer (codec, rng, fit/train/monotone, predict,
 * bucket_index, SplitterTree, duplicate_fraction, verify) is pinned bit-exact
 * against the reference compiled from /root/reference (oracle/_ref, see
 * oracle/Makefile) and against the committed golden vectors in tests/golden/.
 * The sort driver has no reference code; its output is
 * pinned by std::sort / numpy.sort (a keys-only sorted array is unique).
 */
#ifndef LSORT_ORACLE_H
#define LSORT_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LSO_MAX_TREE 1024 /* max bucket budget for a splitter tree */

/* ---- keys.hpp ---------------------------------------------------------- */
uint64_t lso_encode_double(double x);                       /* keys.hpp:24-27 */
double lso_decode_double(uint64_t k);                       /* keys.hpp:29-32 */
int64_t lso_encode_doubles(const double* in, uint64_t* out, size_t n); /* :36-42 */
void lso_decode_doubles(const uint64_t* in, double* out, size_t n);    /* :44-46 */

/* ---- rng.hpp ----------------------------------------------------------- */
uint64_t lso_splitmix64(uint64_t x);                        /* rng.hpp:13-18 */
/* Rng(seed) draw number `draw` (counter-based: splitmix64(seed + draw)). */
uint64_t lso_rng_u64(uint64_t seed, uint64_t draw);         /* rng.hpp:24 */
double lso_rng_unit(uint64_t seed, uint64_t draw);          /* rng.hpp:27-29 */
double lso_rng_unit_open(uint64_t seed, uint64_t draw);     /* rng.hpp:32 */
uint64_t lso_rng_below(uint64_t seed, uint64_t draw, uint64_t bound); /* :35-37 */
double lso_rng_normal(uint64_t seed, uint64_t draw);        /* rng.hpp:41-45, uses draws draw, draw+1 */
double lso_rng_exponential(uint64_t seed, uint64_t draw, double lambda); /* :47-49 */

/* ---- models.hpp / models.cpp: RMI -------------------------------------- */
/* Packed RMI parameters (same layout as lsort_rmi_header/lsort_rmi_entry in
 * include/lsort_cuda.h): P[0]=root.slope P[1]=root.intercept P[2]=key_base
 * P[3]=key_scale, then for m in [0,B): P[4+4m..4m+7] = slope, intercept,
 * clamp_lo, clamp_hi. Size 4+4B doubles. */
int lso_rmi_train(const uint64_t* sorted, size_t n, uint32_t B, double* P); /* models.cpp:39-73 */
/* test hook: train with a caller-provided root (P[0], P[1]) */
int lso_rmi_train_given_root(const uint64_t* sorted, size_t n, uint32_t B, double* P);
void lso_enforce_monotonic(double* P, uint32_t B, const uint64_t* sorted, size_t n); /* models.cpp:75-131 */
double lso_rmi_predict(const double* P, uint32_t B, uint64_t x);    /* models.hpp:34-43 */
uint32_t lso_rmi_route(const double* P, uint32_t B, double xn);     /* models.hpp:60-65 */
uint32_t lso_learned_bucket(const double* P, uint32_t B, uint32_t bucket_count,
                            double cdf_lo, double cdf_hi, uint64_t x); /* models.hpp:162-171 */

/* ---- SplitterTree ------------------------------------------------------ */
typedef struct lso_tree {
    uint32_t levels, leaf_origin, nsplitters, bucket_count;
    uint64_t tree[LSO_MAX_TREE];           /* implicit heap, 1-based, size leaf_origin */
    uint64_t splitters[LSO_MAX_TREE];      /* strictly increasing */
    uint32_t eq_offset[LSO_MAX_TREE + 1];  /* base region -> first bucket id */
} lso_tree;
int lso_tree_build(const uint64_t* sorted, size_t n, uint32_t budget, int equality_mode,
                   lso_tree* t);                                    /* models.cpp:133-185 */
uint32_t lso_tree_classify(const lso_tree* t, uint64_t x);
void lso_learned_bucket_many(const double* P, uint32_t B, uint32_t bucket_count, double cdf_lo, double cdf_hi,
                             const uint64_t* x, size_t n, uint32_t* out);
void lso_tree_classify_many(const lso_tree* t, const uint64_t* x, size_t n, uint32_t* out);          /* models.hpp:92-101 */
double lso_duplicate_fraction(const uint64_t* sorted, size_t n);    /* models.cpp:187-193 */

/* ---- verify.hpp -------------------------------------------------------- */
/* returns 1 if sorted (first_violation=0) else 0 with the index i, a[i-1]>a[i] */
int lso_verify_sorted(const uint64_t* a, size_t n, uint64_t* first_violation); /* verify.hpp:17-22 */
uint64_t lso_multiset_hash(const uint64_t* a, size_t n);           /* verify.hpp:25-29 */

/* ---- synthetic inputs (BASELINE.json configs) ---------- */
enum {
    LSO_GEN_UNIFORM = 0,      /* C1: next_unit, draw i */
    LSO_GEN_NORMAL = 1,       /* C2: next_normal, draws 2i,2i+1 */
    LSO_GEN_LOGNORMAL05 = 2,  /* C2: exp(0.5*normal) */
    LSO_GEN_EXPONENTIAL2 = 3, /* C2: next_exponential(2), draw i */
    LSO_GEN_MIXGAUSS = 4,     /* C3: 5 gaussians, 10 param draws then 3 per element */
    LSO_GEN_ROOTDUPS = 5,     /* C4 (u64): i mod floor(sqrt(N)), Fisher-Yates shuffled */
    LSO_GEN_TWODUPS = 6,      /* C4 (u64): (i*i + N/2) mod N, shuffled */
    LSO_GEN_ZIPF = 7,         /* C4 (u64): Zipf(0.75) over 1e6 ranks, shuffled */
    LSO_GEN_LOGNORMAL2 = 8    /* C5: exp(2*normal) */
};
int lso_gen_is_float(int dist);
/* Elements [first, first+count) of the length-`total` dataset into out
 * (double* for float datasets, uint64_t* otherwise). Shuffled datasets need
 * first == 0 and count == total. */
int lso_generate(int dist, uint64_t total, uint64_t seed, uint64_t first, uint64_t count,
                 void* out, int threads);

/* ---- sort driver (Alg. 5) ------------ */
typedef struct lso_cfg {
    uint32_t rmi_bucket_count;       /* SPEC.md:370  1024 */
    uint32_t tree_bucket_count;      /* 256 */
    uint64_t min_rmi_input;          /* 100000 */
    double max_duplicate_fraction;   /* 0.10 */
    uint32_t radix_base_case;        /* 4096 */
    uint32_t insertion_base_case;    /* 16 */
    uint32_t first_sample_cap;       /* 2*tree_bucket_count*16 */
    uint32_t rmi_sample_cap;         /* 1<<20 */
    double sample_fraction;          /* 0.01 */
    uint64_t seed;
    uint32_t workers;                /* OpenMP threads (0 = all) */
} lso_cfg;
void lso_cfg_default(lso_cfg* c);
uint64_t lso_seg_seed(uint64_t cfg_seed, uint64_t seg_begin, uint32_t depth);
uint64_t lso_first_sample_size(const lso_cfg* c, uint64_t n);
uint64_t lso_rmi_sample_size(const lso_cfg* c, uint64_t n);

/* Alg. 5 build_partition_model for segment a[0,n) that
 * begins at absolute position seg_begin at recursion depth `depth`.
 * kind_out: 0 learned, 1 tree. For learned, P (4+4*rmi_buckets doubles) is
 * filled; for tree, *tree. dup_out = duplicate fraction of the first sample.
 * Sample j of the segment stream is splitmix64(seg_seed + j) % n: the first
 * sample uses j in [0,s1), the RMI sample j in [s1, s1+s2). */
int lso_build_partition_model(const uint64_t* a, uint64_t n, uint64_t seg_begin, uint32_t depth,
                              const lso_cfg* c, uint32_t rmi_buckets, uint32_t tree_buckets,
                              int* kind_out, double* P, lso_tree* tree, double* dup_out);

/* In-place sort of encoded keys (AIPS2o restatement; out-of-place scratch
 * internally). Returns 0. */
int lso_sort_keys(uint64_t* a, uint64_t n, const lso_cfg* c);
/* LearnedSort 2.0 classic path */
void lso_model_counting_sort(const uint64_t* a, size_t n, const double* P, uint32_t B, double cdf_lo,
                             double cdf_hi, uint64_t* out);
int lso_learned_sort_classic(uint64_t* a, uint64_t n, const lso_cfg* c, uint64_t* stats);
/* double entry: encode (NaN -> returns 2, *nan_index set, array untouched),
 * sort, decode. */
int lso_sort_doubles(double* a, uint64_t n, const lso_cfg* c, int64_t* nan_index);

/* ---- pivot analysis -------- */
/* Alg. 4 learned_pivots_for_samplesort: for every key, g = the learned bucket
 * of F(key) with b buckets (models.hpp:162-171, cdf range [0,1]); the pivot
 * for boundary (i+1)/b is the largest key of cell i, i in [0, b-2]; cells
 * never hit are dropped (Alg. 4 "p.filter(v >= 0)"); output strictly
 * increasing. Returns the pivot count (<= b-1); out holds b-1 keys. */
size_t lso_learned_pivots(const uint64_t* a, size_t n, const double* P, uint32_t B, uint32_t b, uint64_t* out);
/* P(A <= p) * N: number of keys <= p in the sorted array (upper bound) */
uint64_t lso_rank_le(const uint64_t* sorted, size_t n, uint64_t p);
/* pivot_quality: sum_{i<np} |P(A <= p_i) - (i+1)/b| (summed in
 * pivot order). Returns -1.0 when np + 1 != b (the metric is defined
 * against b). */
double lso_pivot_quality(const uint64_t* sorted, size_t n, const uint64_t* pivots, size_t np, uint32_t b);
/* eta(pivot) = max(P(A <= p), 1 - P(A <= p)) - 1/2 (§3.1) */
double lso_eta(const uint64_t* sorted, size_t n, uint64_t pivot);

/* radix_base_case_sort: MSD byte radix, insertion <= 16 */
void lso_radix_base_case_sort(uint64_t* a, uint64_t n, uint32_t insertion_threshold);

#ifdef __cplusplus
}
#endif
#endif
