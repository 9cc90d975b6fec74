// ref_capi.cpp -- CPU ORACLE harness (test infrastructure only).
//
// extern "C" wrappers around the reference's own model layer, compiled from
// the unmodified sources under /root/reference/proj/src (see Makefile). The
// resulting oracle/_ref/libref.so is used by tests/ to pin the C restatement
// (lsort_oracle.c) and to generate tests/golden/ fixtures. Nothing in the
// product links it.
#include "keys.hpp"
#include "models.hpp"
#include "rng.hpp"
#include "verify.hpp"

#include <cstring>
#include <stdexcept>

using namespace lsort;

extern "C" {

uint64_t ref_encode_double(double x) { return encode_double(x); }
double ref_decode_double(uint64_t k) { return decode_double(k); }
int64_t ref_encode_doubles(const double* in, uint64_t* out, size_t n) {
    return (int64_t)encode_doubles(in, out, n);
}
uint64_t ref_splitmix64(uint64_t x) { return splitmix64(x); }

// Draw `count` values of kind from Rng(seed) in call order (the reference
// object's own stream): 0 u64, 1 unit, 2 unit_open, 3 below(bound),
// 4 normal, 5 exponential(lambda).
void ref_rng_stream(uint64_t seed, int kind, uint64_t bound, double lambda, size_t count,
                    double* out_d, uint64_t* out_u) {
    Rng r(seed);
    for (size_t i = 0; i < count; ++i) {
        switch (kind) {
        case 0: out_u[i] = r.next_u64(); break;
        case 1: out_d[i] = r.next_unit(); break;
        case 2: out_d[i] = r.next_unit_open(); break;
        case 3: out_u[i] = r.next_below(bound); break;
        case 4: out_d[i] = r.next_normal(); break;
        default: out_d[i] = r.next_exponential(lambda); break;
        }
    }
}

// Packed layout as lsort_oracle.h: P[0..3] root.slope, root.intercept,
// key_base, key_scale; P[4+4m..] slope, intercept, clamp_lo, clamp_hi.
// key_base/key_scale are private in Rmi (models.hpp:71-72); recomputed from
// the sample exactly as models.cpp:47-49 does.
int ref_rmi_train(const uint64_t* s, size_t n, uint32_t B, double* P) {
    try {
        Rmi r = Rmi::train(std::span<const Key>(s, n), B);
        double base = static_cast<double>(s[0]);
        double kmax = static_cast<double>(s[n - 1]);
        P[0] = r.root().slope;
        P[1] = r.root().intercept;
        P[2] = base;
        P[3] = kmax > base ? 1.0 / (kmax - base) : 0.0;
        for (uint32_t m = 0; m < B; ++m) {
            P[4 + 4 * m + 0] = r.submodel(m).slope;
            P[4 + 4 * m + 1] = r.submodel(m).intercept;
            P[4 + 4 * m + 2] = r.clamp_lo(m);
            P[4 + 4 * m + 3] = r.clamp_hi(m);
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// Train, then evaluate predict and PartitionModel::bucket_index on keys.
int ref_rmi_eval(const uint64_t* s, size_t n, uint32_t B, uint32_t bucket_count, double cdf_lo,
                 double cdf_hi, const uint64_t* keys, size_t nk, double* pred, uint32_t* bucket) {
    try {
        Rmi r = Rmi::train(std::span<const Key>(s, n), B);
        PartitionModel pm = PartitionModel::learned(r, bucket_count, cdf_lo, cdf_hi);
        for (size_t i = 0; i < nk; ++i) {
            if (pred) pred[i] = r.predict(keys[i]);
            if (bucket) bucket[i] = pm.bucket_index(keys[i]);
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// SplitterTree::build + classify + exported splitters / equality flags.
int ref_tree_eval(const uint64_t* s, size_t n, uint32_t budget, int eq_mode, const uint64_t* keys,
                  size_t nk, uint32_t* bucket, uint64_t* splitters, uint8_t* heavy,
                  uint32_t* nsplit, uint32_t* bucket_count) {
    try {
        SplitterTree t = SplitterTree::build(std::span<const Key>(s, n), budget, eq_mode != 0);
        PartitionModel pm = PartitionModel::tree(t);
        for (size_t i = 0; i < nk; ++i) bucket[i] = pm.bucket_index(keys[i]);
        *nsplit = (uint32_t)t.splitter_count();
        *bucket_count = t.bucket_count();
        for (size_t i = 0; i < t.splitter_count(); ++i) {
            splitters[i] = t.splitters()[i];
            heavy[i] = t.splitter_has_equality_bucket(i) ? 1 : 0;
        }
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

double ref_duplicate_fraction(const uint64_t* s, size_t n) {
    return duplicate_fraction(std::span<const Key>(s, n));
}

int ref_verify_sorted(const uint64_t* a, size_t n, uint64_t* fv) {
    VerifyResult v = verify_sorted(std::span<const Key>(a, n));
    *fv = v.first_violation;
    return v.sorted ? 1 : 0;
}
uint64_t ref_multiset_hash(const uint64_t* a, size_t n) {
    return multiset_hash(std::span<const Key>(a, n));
}

}  // extern "C"
